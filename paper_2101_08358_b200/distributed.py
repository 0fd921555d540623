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


class DistributedTrainer:
    """train_epoch_partitioned over `world` ranks with the round schedule.

    backend: the rank's step/tables (GpuBackend, or a test backend); dist: torch.distributed,
    initialised by the caller (nccl on GPUs, gloo on CPU)."""

    def __init__(self, backend, num_partitions: int, offsets, batch_size: int, rank: int, world: int,
                 relations: bool, dist=None, group=None):
        if dist is None:
            import torch.distributed as dist
        self.dist, self.group = dist, group
        self.be = backend
        self.rank, self.world = rank, world
        self.plan = make_rounds(num_partitions, world)
        self.offsets = np.asarray(offsets, dtype=np.uint64)
        self.b = batch_size
        self.relations = relations
        # per round: every rank's batch list (all ranks compute all lists: no coordination needed)
        self.batches = [[round_batches(self.plan, self.offsets, batch_size, r, g) for g in range(world)]
                        for r in range(self.plan.rounds)]
        self.steps_per_round = [max(len(x) for x in self.batches[r]) for r in range(self.plan.rounds)]
        self.handoff_bytes = 0

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
        """Lockstep steps [start, start+count) of the epoch (handoffs included when a round ends).
        Returns the number of real edges this rank trained."""
        edges = 0
        for step in range(start, start + count):
            r, s = self.locate(step)
            edges += self._step(r, s, epoch)
            if s + 1 == self.steps_per_round[r]:
                self.handoff(r)
        return edges

    def train_epoch(self, epoch: int) -> dict:
        n = self.run_steps(0, self.total_steps(), epoch)
        return {"edges": n, "steps": self.total_steps(), "handoff_bytes": self.handoff_bytes}

    def _step(self, r: int, s: int, epoch: int) -> int:
        mine = self.batches[r][self.rank]
        n = 0
        if s < len(mine):
            pos, i, j, k, lo, hi, begin, nb = mine[s]
            self.be.train_batch(pos, i, j, k, lo, hi, begin, nb, epoch)
            n = nb
        elif self.relations:
            self.be.zero_relation_grad()  # idle step: contributes nothing to the sum
        if self.relations:
            with self.be.collective_stream():
                self.dist.all_reduce(self.be.relation_grad(), group=self.group)
            self.be.apply_relations()
        return n

    def seek(self, step: int):
        """Positions the partitions for lockstep step `step` of an epoch (from the round-0 layout):
        the partitions move straight to their holders of that step's round."""
        r, _ = self.locate(step)
        if r:
            self.handoff(0, to=r)

    def handoff(self, r: int, to: int | None = None):
        """Partitions leaving this rank after round r go to their round-(r+1) (or round-`to`) holder
        (P2P: NCCL over NVLink for device tensors; a gloo group moves device tables through host
        copies)."""
        moves = self.plan.transfers(r, to)
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
