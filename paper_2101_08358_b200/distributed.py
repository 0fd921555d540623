"""Multi-GPU partitioned training: one process per GPU, buckets in conflict-free rounds.

The path shards at bucket granularity: bucket (i, j) touches node partitions i and j and the
(small, replicated) relation table only (Algorithm 2). Each round of
`make_rounds` (csrc/host/rounds.cpp) is a perfect matching of the p partitions, so no partition is
on two GPUs at once; between rounds a partition moves to its next holder by a point-to-point
send (NCCL over NVLink on B200, gloo in the CPU tests). Only the relation gradients are summed
across ranks, every step, before the relation Adagrad (SPEC.md:388 synchronous relations; the
reduced bytes are identical on every rank, so the relation replicas stay bit-identical).

Lockstep: the relation all-reduce is a collective, so every rank takes the same number of steps
per round: max over ranks of the round's batch count. A rank whose buckets are exhausted takes
an idle step (zero relation gradient, same all-reduce and Adagrad). Dot models have no relations
and need no per-step collective at all (only the round handoffs).

The per-rank step is a backend: `GpuBackend` calls the C-ABI on the rank's GPU (the product);
the CPU tests plug in a backend over the oracle to check this orchestration with gloo.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from ._lib import check, lib


def check_or(status: int, trainer) -> int:
    """check() for ember_dist_run: an exception raised inside a callback is re-raised as itself."""
    if status and getattr(trainer, "_error", None) is not None:
        err, trainer._error = trainer._error, None
        raise err
    check(status)
    return status


@dataclass
class RoundPlan:
    """make_rounds(p, world): the global bucket schedule and who holds which partition when."""
    p: int
    world: int
    rounds: int
    order: np.ndarray   # [p*p] bucket ids i*p+j in global schedule order (position = bucket_step)
    round: np.ndarray   # [p*p] round of each position
    rank: np.ndarray    # [p*p] GPU of each position
    holder: np.ndarray  # [rounds, p] GPU holding partition x during round r
    early: np.ndarray | None = None  # [p*p] overlapped schedule: bucket's partitions leave after the round

    def buckets(self, r: int, g: int) -> list[tuple[int, int, int]]:
        """(bucket_step, i, j) of GPU g in round r, in training order."""
        sel = np.nonzero((self.round == r) & (self.rank == g))[0]
        return [(int(s), int(self.order[s]) // self.p, int(self.order[s]) % self.p) for s in sel]

    def partitions(self, r: int, g: int) -> list[int]:
        return [int(x) for x in np.nonzero(self.holder[r] == g)[0]]

    def transfers(self, r: int, to: int | None = None) -> list[tuple[int, int, int]]:
        """(partition, src, dst) moving between round r and round `to` (default: the next one; the
        last round hands over to round 0 of the next epoch), ascending partition."""
        a, b = self.holder[r], self.holder[(r + 1) % self.rounds if to is None else to]
        return [(int(x), int(a[x]), int(b[x])) for x in range(self.p) if a[x] != b[x]]


def make_rounds(p: int, world: int, overlap: bool = False) -> RoundPlan:
    """Circle-method rounds (ember_make_rounds), or with overlap=True the coset schedule
    (ember_make_rounds_overlap: p a power of two, world | p/4) whose departing partitions are used
    only by each round's first (early) buckets."""
    n = p * p
    order, rnd, rank = (np.zeros(n, np.uint32) for _ in range(3))
    holder = np.zeros(max(1, p - 1) * p, np.uint32)
    nr = C.c_uint32(0)
    early = None
    if overlap:
        early = np.zeros(n, np.uint8)
        check(lib().ember_make_rounds_overlap(p, world, order.ctypes.data, rnd.ctypes.data, rank.ctypes.data,
                                              early.ctypes.data, holder.ctypes.data, C.byref(nr)))
    else:
        check(lib().ember_make_rounds(p, world, order.ctypes.data, rnd.ctypes.data, rank.ctypes.data,
                                      holder.ctypes.data, C.byref(nr)))
    R = int(nr.value)
    return RoundPlan(p, world, R, order, rnd, rank, holder[:R * p].reshape(R, p), early)


def round_batches(plan: RoundPlan, offsets, batch_size: int, r: int, g: int) -> list[tuple]:
    """Batches of GPU g in round r: (bucket_step, i, j, batch_in_bucket, lo, hi, begin, nb);
    the bucket's edges are [lo, hi) of the bucketed edge array, the batch [lo+begin, +nb)."""
    out = []
    for s, i, j in plan.buckets(r, g):
        b = i * plan.p + j
        lo, hi = int(offsets[b]), int(offsets[b + 1])
        for k, b0 in enumerate(range(lo, hi, batch_size)):
            out.append((s, i, j, k, lo, hi, b0 - lo, min(batch_size, hi - b0)))
    return out


class _BatchRef(C.Structure):
    _fields_ = [("bucket_step", C.c_uint32), ("i", C.c_uint32), ("j", C.c_uint32), ("batch_in_bucket", C.c_uint32),
                ("lo", C.c_uint64), ("hi", C.c_uint64), ("begin", C.c_uint64), ("nb", C.c_uint32), ("pad", C.c_uint32)]


_STEP = C.CFUNCTYPE(C.c_int, C.c_void_p, C.POINTER(_BatchRef), C.c_uint64)
_SEND_RECV = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_uint32, C.POINTER(C.c_uint32), C.c_uint32)
_ACQUIRE = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_uint32, C.POINTER(C.c_uint32), C.c_uint32)


class _RankOps(C.Structure):
    _fields_ = [("user", C.c_void_p), ("step", _STEP), ("send_recv", _SEND_RECV), ("acquire", _ACQUIRE)]


class DistReport(C.Structure):
    _fields_ = [(f, C.c_uint64) for f in ("steps", "batches", "edges", "handoffs", "moved_partitions",
                                          "early_handoffs", "handoff_bytes")]


class DistributedTrainer:
    """train_epoch_partitioned over `world` ranks with the round schedule.

    The round loop is the library's (host C++, csrc/host/dist_driver.cpp, ember_dist_run): it calls
    back into this object for each lockstep step (the backend's batch or an idle step, then the
    relation all-reduce through torch.distributed) and at each handoff point (P2P through
    torch.distributed). backend: the rank's step/tables (GpuBackend, or a test backend); dist:
    torch.distributed, initialised by the caller (nccl on GPUs, gloo on CPU). The all-native GPU
    form (NCCL inside the library, copies on their own stream) is ember_dist_create / NativeDistributed.
    overlap: the coset schedule (make_rounds(..., overlap=True))."""

    def __init__(self, backend, num_partitions: int, offsets, batch_size: int, rank: int, world: int,
                 relations: bool, dist=None, group=None, overlap: bool = False):
        if dist is None:
            import torch.distributed as dist
        self.dist, self.group = dist, group
        self.be = backend
        self.rank, self.world = rank, world
        self.overlap = bool(overlap)
        self.plan = make_rounds(num_partitions, world, overlap=self.overlap)
        self.offsets = np.ascontiguousarray(np.asarray(offsets, dtype=np.uint64))
        self.b = batch_size
        self.relations = relations
        R = self.plan.rounds
        steps, hand = np.zeros(R, np.uint32), np.zeros(R, np.uint32)
        total = C.c_uint64(0)
        check(lib().ember_dist_plan(num_partitions, world, rank, int(self.overlap), self.offsets.ctypes.data,
                                    batch_size, steps.ctypes.data, hand.ctypes.data, C.byref(total)))
        self.steps_per_round = [int(x) for x in steps]
        self.handoff_step = [int(x) for x in hand]
        self.handoff_bytes = 0
        self.report = DistReport()
        self._error = None

    # -- setup --------------------------------------------------------------------------------
    def init_embeddings(self, seed: int):
        """init_embeddings of this rank's round-0 partitions + the relation replica:
        per global row, so the union over ranks equals a 1-GPU init bit for bit."""
        for x in self.plan.partitions(0, self.rank):
            self.be.init_partition(x, seed)
        self.be.init_relations(seed)

    # -- the epoch ------------------------------------------------------------------------------
    def total_steps(self) -> int:
        return sum(self.steps_per_round)

    def locate(self, step: int) -> tuple[int, int]:
        """Global lockstep step -> (round, step within round)."""
        for r, n in enumerate(self.steps_per_round):
            if step < n:
                return r, step
            step -= n
        raise IndexError("step beyond the epoch")

    def run_steps(self, start: int, count: int, epoch: int) -> int:
        """Lockstep steps [start, start+count) of the epoch through the library's round loop (handoffs
        included where the schedule puts them). Returns the number of real edges this rank trained."""
        def guard(fn):
            def wrapped(*a):
                try:
                    fn(*a)
                    return 0
                except BaseException as ex:  # surfaced after the C call returns
                    self._error = ex
                    return 1
            return wrapped

        def step(_, bp, ep):
            self._step(bp.contents if bp else None, int(ep))

        def send_recv(_, r, mv, n):
            self._send_recv([(int(mv[3 * k]), int(mv[3 * k + 1]), int(mv[3 * k + 2])) for k in range(n)])

        ops = _RankOps(None, _STEP(guard(step)), _SEND_RECV(guard(send_recv)), _ACQUIRE(0))
        rep = DistReport()
        self._error = None
        check_or(lib().ember_dist_run(self.plan.p, self.world, self.rank, int(self.overlap), self.offsets.ctypes.data,
                                      self.b, epoch, start, count, C.byref(ops), C.byref(rep)), self)
        for f, _ in DistReport._fields_:
            setattr(self.report, f, getattr(self.report, f) + getattr(rep, f))
        return int(rep.edges)

    def train_epoch(self, epoch: int) -> dict:
        n = self.run_steps(0, self.total_steps(), epoch)
        return {"edges": n, "steps": self.total_steps(), "handoff_bytes": self.handoff_bytes}

    def _step(self, b, epoch: int):
        if b is not None:
            self.be.train_batch(b.bucket_step, b.i, b.j, b.batch_in_bucket, b.lo, b.hi, b.begin, b.nb, epoch)
        elif self.relations:
            self.be.zero_relation_grad()  # idle step: contributes nothing to the sum
        if self.relations:
            with self.be.collective_stream():
                self.dist.all_reduce(self.be.relation_grad(), group=self.group)
            self.be.apply_relations()

    def seek(self, step: int):
        """Positions the partitions for lockstep step `step` of an epoch (from the round-0 layout):
        the partitions move straight to their holders of that step's round."""
        r, _ = self.locate(step)
        if r:
            self.handoff(0, to=r)

    def handoff(self, r: int, to: int | None = None):
        """Partitions leaving this rank after round r go to their round-(r+1) (or round-`to`) holder."""
        self._send_recv(self.plan.transfers(r, to))

    def _send_recv(self, moves):
        """This rank's part of one handoff (P2P: NCCL over NVLink for device tensors; a gloo group
        moves device tables through host copies)."""
        if not moves:
            return
        ops, incoming = [], []
        P2P = self.dist.P2POp
        stage = self._host_staged()
        with self.be.collective_stream():
            for x, src, dst in moves:
                if src == self.rank:
                    th, ac = self.be.tables(x)
                    if stage:
                        th, ac = th.cpu(), ac.cpu()
                    ops += [P2P(self.dist.isend, th, dst, self.group), P2P(self.dist.isend, ac, dst, self.group)]
                    self.handoff_bytes += th.numel() * th.element_size() * 2
                elif dst == self.rank:
                    th, ac = self.be.empty_tables(x)
                    bufs = (th.cpu(), ac.cpu()) if stage else (th, ac)
                    ops += [P2P(self.dist.irecv, bufs[0], src, self.group),
                            P2P(self.dist.irecv, bufs[1], src, self.group)]
                    incoming.append((x, th, ac, bufs))
            if ops:
                for w in self.dist.batch_isend_irecv(ops):
                    w.wait()
            if stage:
                for x, th, ac, bufs in incoming:
                    th.copy_(bufs[0])
                    ac.copy_(bufs[1])
        self.be.after_handoff()
        for x, src, dst in moves:
            if src == self.rank:
                self.be.drop(x)
        for x, th, ac, _ in incoming:
            self.be.adopt(x, th, ac)

    def _host_staged(self) -> bool:
        try:
            backend = self.dist.get_backend(self.group)
        except Exception:
            return False
        return backend == "gloo" and getattr(self.be, "device_tables", False)

    def local_tables(self):
        """This rank's partitions between epochs (the round-0 holders), as {x: (theta, acc)}."""
        return {x: self.be.tables(x) for x in self.plan.partitions(0, self.rank)}


class GpuBackend:
    """The rank's GPU: a Trainer (C-ABI context) whose partition tables are bound as they arrive,
    relation gradients reduced externally (ember_relations_external) by the trainer's all-reduce on
    the context stream."""

    device_tables = True

    def __init__(self, trainer, edges_dev):
        import torch
        self.torch = torch
        self.tr = trainer
        self.edges = edges_dev
        self.base = edges_dev.data_ptr()
        self.tabs: dict[int, tuple] = {}
        h = trainer.h
        self.rel_grad = None
        if trainer.rel_theta is not None:
            self.rel_grad = torch.zeros((trainer.R, h.dim), dtype=torch.float32, device=trainer.dev)
            check(lib().ember_relations_external(trainer.ctx, self.rel_grad.data_ptr()))
        self.stream = trainer.torch_stream()
        # e2e mode: positives come from pinned host memory (ember_train_batch_host), loss read back
        self.host_edges = None
        self.loss_host = None
        self.h2d_bytes = 0

    def _rows(self, x):
        from . import partition_size
        return partition_size(self.tr.V, self.tr.p, x)

    def empty_tables(self, x):
        t = self.torch
        with t.cuda.stream(self.stream):
            return (t.empty((self._rows(x), self.tr.h.dim), dtype=t.float32, device=self.tr.dev),
                    t.empty((self._rows(x), self.tr.h.dim), dtype=t.float32, device=self.tr.dev))

    def init_partition(self, x, seed):
        th, ac = self.empty_tables(x)
        self.adopt(x, th, ac)
        check(lib().ember_init_partition(self.tr.ctx, x, seed))

    def init_relations(self, seed):
        if self.tr.rel_theta is not None:
            check(lib().ember_init_relations(self.tr.ctx, seed))

    def adopt(self, x, th, ac):
        self.tabs[x] = (th, ac)
        check(lib().ember_tables_bind(self.tr.ctx, x, th.data_ptr(), ac.data_ptr()))

    def drop(self, x):
        self.tabs.pop(x, None)

    def tables(self, x):
        return self.tabs[x]

    def train_batch(self, pos, i, j, k, lo, hi, begin, nb, epoch):
        if self.host_edges is None:
            check(lib().ember_train_batch(self.tr.ctx, self.base + 12 * lo, hi - lo, begin, nb, i, j, epoch, pos, k,
                                          None))
        else:
            check(lib().ember_train_batch_host(self.tr.ctx, self.base + 12 * lo, hi - lo,
                                               self.host_edges.data_ptr() + 12 * (lo + begin), nb, i, j, epoch, pos,
                                               k, self.loss_host.data_ptr()))
            self.h2d_bytes += 12 * nb

    def zero_relation_grad(self):
        with self.torch.cuda.stream(self.stream):
            self.rel_grad.zero_()

    def relation_grad(self):
        return self.rel_grad

    def apply_relations(self):
        check(lib().ember_relations_apply_dense(self.tr.ctx, self.rel_grad.data_ptr()))

    def collective_stream(self):
        return self.torch.cuda.stream(self.stream)

    def after_handoff(self):
        # sent buffers may be released only once their sends have completed
        self.stream.synchronize()


def nccl_unique_id() -> bytes:
    """A fresh ncclUniqueId (128 bytes; rank 0 makes it, the caller shares it, e.g. by broadcast)."""
    buf = C.create_string_buffer(128)
    check(lib().ember_nccl_unique_id(buf))
    return buf.raw


class NativeDistributed:
    """train_epoch_partitioned over `world` GPUs entirely in the library (ember_dist_*): the C++ round
    loop, the NCCL relation all-reduce on the step stream and the NCCL P2P partition handoffs on a
    copy stream with a second communicator. The driver owns the node tables, so `trainer` is created
    with allocate=False (its relation replica stays bound). ids: two ncclUniqueId (bytes) shared by
    the ranks, None at world 1."""

    def __init__(self, trainer, edges_dev, offsets, rank: int, world: int, overlap: bool = True,
                 ids: tuple[bytes, bytes] | None = None):
        self.tr, self.edges = trainer, edges_dev
        self.offsets = np.ascontiguousarray(np.asarray(offsets, dtype=np.uint64))
        self.rank, self.world, self.overlap = rank, world, bool(overlap)
        a = b = None
        if world > 1:
            if ids is None:
                raise ValueError("world > 1 needs two NCCL unique ids")
            a, b = C.create_string_buffer(ids[0], 128), C.create_string_buffer(ids[1], 128)
        h = C.c_void_p()
        trainer._enter(edges_dev)
        check(lib().ember_dist_create(trainer.ctx, rank, world, int(self.overlap), a, b, edges_dev.data_ptr(),
                                      self.offsets.ctypes.data, C.byref(h)))
        self.h = h
        self.plan = make_rounds(trainer.p, world, overlap=self.overlap)
        R = self.plan.rounds
        steps, hand = np.zeros(R, np.uint32), np.zeros(R, np.uint32)
        total = C.c_uint64(0)
        check(lib().ember_dist_plan(trainer.p, world, rank, int(self.overlap), self.offsets.ctypes.data,
                                    trainer.h.batch_size, steps.ctypes.data, hand.ctypes.data, C.byref(total)))
        self.steps_per_round = [int(x) for x in steps]
        self.handoff_step = [int(x) for x in hand]

    def total_steps(self) -> int:
        return sum(self.steps_per_round)

    def init_embeddings(self, seed: int):
        check(lib().ember_dist_init_embeddings(self.h, seed))

    def run_steps(self, start: int, count: int, epoch: int) -> DistReport:
        rep = DistReport()
        check(lib().ember_dist_train_epoch(self.h, epoch, start, count, C.byref(rep)))
        return rep

    def train_epoch(self, epoch: int) -> DistReport:
        return self.run_steps(0, 2 ** 64 - 1, epoch)

    def synchronize(self):
        check(lib().ember_dist_synchronize(self.h))

    def loss(self) -> float:
        v = C.c_float(0.0)
        check(lib().ember_dist_loss(self.h, C.byref(v)))
        return float(v.value)

    def held(self) -> list[int]:
        out = []
        for x in range(self.tr.p):
            th = C.c_void_p()
            check(lib().ember_dist_tables(self.h, x, C.byref(th), None))
            if th.value:
                out.append(x)
        return out

    def partition_table(self, x: int):
        """theta/acc of a partition this rank holds: host copies in on-disk coordinate order."""
        from . import partition_size, rows_to_disk
        th, ac = C.c_void_p(), C.c_void_p()
        check(lib().ember_dist_tables(self.h, x, C.byref(th), C.byref(ac)))
        if not th.value:
            raise ValueError(f"partition {x} is not on this rank")
        self.synchronize()
        n = partition_size(self.tr.V, self.tr.p, x) * self.tr.h.dim
        outs = []
        for ptr in (th.value, ac.value):
            a = np.empty(n, np.float32)
            check(lib().ember_copy_to_host(self.tr.ctx, a.ctypes.data, ptr, 4 * n))
            outs.append(rows_to_disk(a.reshape(-1, self.tr.h.dim), self.tr.h.kind))
        return outs[0], outs[1]

    def close(self):
        if getattr(self, "h", None):
            check(lib().ember_dist_destroy(self.h))
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
