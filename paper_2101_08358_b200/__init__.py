"""ember-b200: B200-native minibatch training step of Gaius/Marius (arXiv 2101.08358).

Host mirror of the reference's (reconstructed) model / ordering / pipeline surface over the
C-ABI in include/ember_gpu.h. Device memory is torch-allocated (plumbing); all compute runs in
libember_b200.so (sm_100a). Names follow the reference: ModelKind, OrderingPlan, make_plan,
sample_negatives, loss_and_grad, adagrad_step, init_embeddings, train_epoch_partitioned.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from ._lib import (ENGINE, KIND, ORDERING, BufferReport, ConfigError, EmberError, GraphDesc, ModelDesc,  # noqa: F401
                   StepStats, check, lib)

__all__ = ["ConfigError", "EmberError", "Hyper", "Trainer", "PartitionBuffer", "preprocess_graph", "make_plan", "lower_bound_swaps",
           "elimination_swap_formula", "generate_graph", "bucket_edges", "partition_offset", "partition_size", "lib",
           "rows_to_disk", "rows_to_hbm"]


def partition_offset(V: int, p: int, k: int) -> int:
    q, r = divmod(V, p)
    return k * q + min(k, r)


def partition_size(V: int, p: int, k: int) -> int:
    q, r = divmod(V, p)
    return q + (1 if k < r else 0)


def rows_to_disk(x: np.ndarray, kind) -> np.ndarray:
    """Rows in the HBM row layout -> on-disk coordinate order. Only ComplEx rows
    differ: HBM holds their [re | im] halves interleaved by pairs (include/ember_gpu.h)."""
    x = np.asarray(x)
    if KIND.get(kind, kind) != KIND["complex"]:
        return x
    n, d = x.shape
    return np.ascontiguousarray(x.reshape(n, d // 4, 2, 2).transpose(0, 2, 1, 3).reshape(n, d))


def rows_to_hbm(x: np.ndarray, kind) -> np.ndarray:
    """On-disk coordinate order -> the HBM row layout (inverse of rows_to_disk)."""
    x = np.asarray(x)
    if KIND.get(kind, kind) != KIND["complex"]:
        return x
    n, d = x.shape
    return np.ascontiguousarray(x.reshape(n, 2, d // 4, 2).transpose(0, 2, 1, 3).reshape(n, d))


def _ptr(x) -> int | None:
    if x is None:
        return None
    if hasattr(x, "data_ptr"):
        return x.data_ptr()
    if isinstance(x, np.ndarray):
        return x.ctypes.data
    return int(x)


# ---------------------------------------------------------------------------------- ordering

def make_plan(kind: str | int, p: int, c: int, seed: int = 0) -> dict:
    """make_plan (reference ordering.h:80 / ordering.cpp:384): BETA (elimination), hilbert, ..."""
    k = ORDERING[kind] if isinstance(kind, str) else int(kind)
    seq = np.zeros(2 * p * p, np.uint32)
    adm = np.zeros(c + 2 * p * p + 1, np.uint32)
    swaps = np.zeros(6 * p * p + 3, np.uint32)
    state = np.zeros(p * p, np.uint32)
    sc = C.c_uint64(0)
    na = C.c_uint32(0)
    check(lib().ember_make_plan(k, p, c, seed, _ptr(seq), C.byref(sc), _ptr(adm), C.byref(na), _ptr(swaps),
                                _ptr(state)))
    n = int(sc.value)
    return {"seq": seq.reshape(-1, 2), "swap_count": n, "admissions": adm[: na.value].copy(),
            "swaps": swaps[: 3 * n].reshape(-1, 3).copy(), "bucket_state": state}


def lower_bound_swaps(p: int, c: int) -> int:
    v = lib().ember_lower_bound_swaps(p, c)
    if v == (1 << 64) - 1:
        raise ConfigError(lib().ember_last_error().decode())
    return int(v)


def elimination_swap_formula(p: int, c: int) -> int:
    v = lib().ember_elimination_swap_formula(p, c)
    if v == (1 << 64) - 1:
        raise ConfigError(lib().ember_last_error().decode())
    return int(v)


# ---------------------------------------------------------------------------------- graphs

def generate_graph(num_nodes: int, num_relations: int, n_edges: int, seed: int, train_frac=0.9, valid_frac=0.05,
                   device: int | None = None):
    """Synthetic planted-community graph. device=None -> numpy (host), else torch tensors on cuda:device."""
    if device is None:
        edges = np.zeros((n_edges, 3), np.uint32)
        split = np.zeros(n_edges, np.uint8)
        check(lib().ember_graph_generate(-1, num_nodes, num_relations, n_edges, seed, train_frac, valid_frac,
                                         _ptr(edges), _ptr(split)))
        return edges, split
    import torch
    edges = torch.empty((n_edges, 3), dtype=torch.int32, device=f"cuda:{device}")
    split = torch.empty(n_edges, dtype=torch.uint8, device=f"cuda:{device}")
    check(lib().ember_graph_generate(device, num_nodes, num_relations, n_edges, seed, train_frac, valid_frac,
                                     _ptr(edges), _ptr(split)))
    return edges, split


def bucket_edges(edges, num_nodes: int, p: int, device: int | None = None):
    """bucket_edges: stable sort into p*p buckets; returns (edges, offsets[p*p+1])."""
    n = int(edges.shape[0])
    offsets = np.zeros(p * p + 1, np.uint64)
    if device is None:
        edges = np.ascontiguousarray(edges, np.uint32)
        out = np.zeros_like(edges)
        check(lib().ember_graph_bucket(-1, num_nodes, p, _ptr(edges), n, _ptr(out), _ptr(offsets)))
        return out, offsets
    import torch
    out = torch.empty_like(edges)
    check(lib().ember_graph_bucket(device, num_nodes, p, _ptr(edges), n, _ptr(out), _ptr(offsets)))
    return out, offsets


def preprocess_graph(raw_edges, p: int, seed: int, train_frac: float = 0.9, valid_frac: float = 0.05,
                     device: int = 0) -> dict:
    """Graph-store preprocessing on the device: dense ids, seeded node permutation,
    seeded shuffle + split, stable bucketing of train. raw_edges: (n, 3) u32 tokens (numpy or a
    device tensor). Returns device tensors train/valid/test, offsets (numpy), num_nodes,
    num_relations and the token of every relabeled node / relation id."""
    import torch
    dev = torch.device(f"cuda:{device}")
    raw = raw_edges if hasattr(raw_edges, "data_ptr") else torch.from_numpy(
        np.ascontiguousarray(raw_edges, np.uint32).view(np.int32))
    raw = raw.to(dev).contiguous()
    n = int(raw.shape[0])
    train = torch.empty((n, 3), dtype=torch.int32, device=dev)
    valid = torch.empty((n, 3), dtype=torch.int32, device=dev)
    test = torch.empty((n, 3), dtype=torch.int32, device=dev)
    ntok = torch.empty(2 * n, dtype=torch.int32, device=dev)
    rtok = torch.empty(n, dtype=torch.int32, device=dev)
    offsets = np.zeros(p * p + 1, np.uint64)
    counts = np.zeros(3, np.uint64)
    V, R = C.c_uint64(0), C.c_uint32(0)
    check(lib().ember_graph_preprocess(device, _ptr(raw), n, p, seed, train_frac, valid_frac, _ptr(train),
                                       _ptr(offsets), _ptr(valid), _ptr(test), _ptr(counts), _ptr(ntok), _ptr(rtok),
                                       C.byref(V), C.byref(R)))
    a, b, c = (int(x) for x in counts)
    return {"train": train[:a], "valid": valid[:b], "test": test[:c], "offsets": offsets, "num_nodes": V.value,
            "num_relations": R.value, "node_tokens": ntok[:V.value], "rel_tokens": rtok[:R.value]}


# ---------------------------------------------------------------------------------- trainer

@dataclass
class Hyper:
    """RunConfig subset consumed by the step (Table 1 defaults)."""
    kind: str = "complex"
    dim: int = 100
    lr: float = 0.1
    eps: float = 1e-10
    batch_size: int = 50_000
    num_negatives: int = 1000
    alpha: float = 0.5
    num_chunks: int = 1
    neg_seed: int = 1
    engine: str = "tc"  # "simt": the tests' fp32 reference engine (needs EMBER_TEST_ENGINES=1)

    def desc(self) -> ModelDesc:
        return ModelDesc(KIND[self.kind], self.dim, self.lr, self.eps, self.batch_size, self.num_negatives,
                         self.alpha, self.num_chunks, self.neg_seed, ENGINE[self.engine], 0)


class Trainer:
    """One GPU's training context: partition tables in HBM + the C-ABI step.

    tables: allocate=True allocates theta/acc for every partition on this GPU (torch, fp32) and
    binds them; pass allocate=False to bind externally owned slots with bind_partition().
    """

    def __init__(self, hyper: Hyper, num_nodes: int, num_relations: int, num_partitions: int = 1, device: int = 0,
                 allocate: bool = True, stream=None):
        import torch
        self.torch = torch
        self.h = hyper
        self.V, self.R, self.p = num_nodes, num_relations, num_partitions
        self.device = device
        self.dev = torch.device(f"cuda:{device}")
        md = hyper.desc()
        gd = GraphDesc(num_nodes, num_relations, num_partitions)
        ctx = C.c_void_p()
        if stream is None:
            # a torch-owned stream (torch never destroys its streams): tensors recorded on it with
            # record_stream stay valid after the context is gone; highest priority, like the
            # engine's own stream
            stream = torch.cuda.Stream(device=self.dev, priority=-100)
        self._ts = stream
        check(lib().ember_ctx_create(device, C.byref(md), C.byref(gd), stream.cuda_stream, C.byref(ctx)))
        self.ctx = ctx
        self.theta: dict[int, object] = {}
        self.acc: dict[int, object] = {}
        self.rel_theta = self.rel_acc = None
        if allocate:
            for k in range(num_partitions):
                rows = partition_size(num_nodes, num_partitions, k)
                self.bind_partition(k, torch.empty((rows, hyper.dim), dtype=torch.float32, device=self.dev),
                                    torch.empty((rows, hyper.dim), dtype=torch.float32, device=self.dev))
        if KIND[hyper.kind] != 0:  # relations are always HBM-resident (5.9 MB at FB86m)
            self.bind_relations(torch.empty((num_relations, hyper.dim), dtype=torch.float32, device=self.dev),
                                torch.empty((num_relations, hyper.dim), dtype=torch.float32, device=self.dev))

    # -- lifecycle ------------------------------------------------------------------------
    def close(self):
        if getattr(self, "ctx", None):
            check(lib().ember_ctx_destroy(self.ctx))
            self.ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def stream_ptr(self) -> int:
        return lib().ember_ctx_stream(self.ctx)

    def torch_stream(self):
        return self._ts

    def _enter(self, *tensors):
        """Orders a C-ABI call after the caller's work: the context stream waits for torch's current
        stream (which produced the inputs), and every borrowed device tensor is recorded on the
        context stream, so torch's caching allocator cannot hand its memory out again before the
        engine's (asynchronous) kernels are done with it."""
        t = self.torch
        ts = self.torch_stream()
        cur = t.cuda.current_stream(self.dev)
        if cur.cuda_stream != ts.cuda_stream:
            ts.wait_stream(cur)
        for x in tensors:
            if x is not None and isinstance(x, t.Tensor) and x.is_cuda:
                x.record_stream(ts)

    def _leave(self):
        """Outputs handed back without a host synchronisation: torch's current stream waits for them."""
        t = self.torch
        ts = self.torch_stream()
        cur = t.cuda.current_stream(self.dev)
        if cur.cuda_stream != ts.cuda_stream:
            cur.wait_stream(ts)

    def synchronize(self):
        check(lib().ember_ctx_synchronize(self.ctx))
        self.torch.cuda.synchronize(self.dev)

    # -- tables ---------------------------------------------------------------------------
    def bind_partition(self, k, theta, acc):
        self.theta[k], self.acc[k] = theta, acc
        self._enter(theta, acc)
        check(lib().ember_tables_bind(self.ctx, k, _ptr(theta), _ptr(acc)))

    def bind_relations(self, theta, acc):
        self.rel_theta, self.rel_acc = theta, acc
        self._enter(theta, acc)
        check(lib().ember_relations_bind(self.ctx, _ptr(theta), _ptr(acc)))

    def init_embeddings(self, seed: int):
        """init_embeddings: every bound partition + relations, on the device."""
        self._enter()
        for k in self.theta:
            check(lib().ember_init_partition(self.ctx, k, seed))
        if self.rel_theta is not None:
            check(lib().ember_init_relations(self.ctx, seed))
        self._leave()

    def node_table(self):
        """Concatenated theta/acc of all partitions: host copies in on-disk coordinate order (the
        device tables hold the HBM row layout, rows_to_disk)."""
        self.synchronize()
        th = self.torch.cat([self.theta[k] for k in range(self.p)]).cpu().numpy()
        ac = self.torch.cat([self.acc[k] for k in range(self.p)]).cpu().numpy()
        return rows_to_disk(th, self.h.kind), rows_to_disk(ac, self.h.kind)

    def relation_table(self):
        """theta/acc of the relation table, host copies in on-disk coordinate order."""
        self.synchronize()
        return (rows_to_disk(self.rel_theta.cpu().numpy(), self.h.kind),
                rows_to_disk(self.rel_acc.cpu().numpy(), self.h.kind))

    # -- the step -------------------------------------------------------------------------
    def train_batch(self, bucket_edges, batch_begin: int, nb: int, i: int = 0, j: int = 0, epoch: int = 0,
                    bucket_step: int = 0, batch_in_bucket: int = 0, loss_out=None):
        self._enter(bucket_edges, loss_out)
        check(lib().ember_train_batch(self.ctx, _ptr(bucket_edges), int(bucket_edges.shape[0]), batch_begin, nb, i, j,
                                      epoch, bucket_step, batch_in_bucket, _ptr(loss_out)))
        self._leave()

    def train_batch_host(self, bucket_edges, host_batch, i=0, j=0, epoch=0, bucket_step=0, batch_in_bucket=0,
                         want_loss=True) -> float | None:
        loss = C.c_float(0.0)
        self._enter(bucket_edges)
        check(lib().ember_train_batch_host(self.ctx, _ptr(bucket_edges), int(bucket_edges.shape[0]), _ptr(host_batch),
                                           int(host_batch.shape[0]), i, j, epoch, bucket_step, batch_in_bucket,
                                           C.byref(loss) if want_loss else None))
        if want_loss:
            check(lib().ember_ctx_synchronize(self.ctx))
        return float(loss.value) if want_loss else None

    def train_bucket(self, bucket_edges, i=0, j=0, epoch=0, bucket_step=0) -> StepStats:
        st = StepStats()
        self._enter(bucket_edges)
        check(lib().ember_train_bucket(self.ctx, _ptr(bucket_edges), int(bucket_edges.shape[0]), i, j, epoch,
                                       bucket_step, C.byref(st)))
        return st

    def train_epoch(self, edges_dev, offsets, plan_seq, epoch: int) -> dict:
        """train_epoch_partitioned (Algorithm 2): buckets in plan order, one C-ABI call
        (no host synchronisation inside the epoch)."""
        st = StepStats()
        seq = np.ascontiguousarray(np.asarray(plan_seq, dtype=np.uint32).reshape(-1))
        off = np.ascontiguousarray(np.asarray(offsets, dtype=np.uint64))
        self._enter(edges_dev)
        check(lib().ember_train_epoch(self.ctx, _ptr(edges_dev), _ptr(off), _ptr(seq), epoch, C.byref(st)))
        return {"loss": st.loss_sum / max(1, st.batches), "batches": st.batches, "edges": st.edges}

    # -- per-op entry points (parity tests) ----------------------------------------------
    def sample_negatives(self, bucket_edges, i=0, j=0, epoch=0, bucket_step=0, batch_in_bucket=0):
        t = self.torch
        out = t.empty(max(1, self.h.num_chunks) * 2 * self.h.num_negatives, dtype=t.int32, device=self.dev)
        self._enter(bucket_edges, out)
        check(lib().ember_sample_negatives(self.ctx, _ptr(bucket_edges), int(bucket_edges.shape[0]), i, j, epoch,
                                           bucket_step, batch_in_bucket, _ptr(out)))
        self._leave()
        return out

    def loss_and_grad(self, edges, negs, i=0, j=0) -> dict:
        t = self.torch
        nb = int(edges.shape[0])
        d = self.h.dim
        cap = 2 * nb + int(negs.numel())
        fpos = t.empty(nb, dtype=t.float32, device=self.dev)
        lse = t.empty(2 * nb, dtype=t.float32, device=self.dev)
        ids = t.empty(cap, dtype=t.int32, device=self.dev)
        rows = t.empty((cap, d), dtype=t.float32, device=self.dev)
        rids = t.empty(max(nb, 1), dtype=t.int32, device=self.dev)
        rrows = t.empty((max(nb, 1), d), dtype=t.float32, device=self.dev)
        nu, nr, loss = C.c_uint32(0), C.c_uint32(0), C.c_double(0)
        self._enter(edges, negs, fpos, lse, ids, rows, rids, rrows)
        check(lib().ember_loss_and_grad(self.ctx, _ptr(edges), nb, i, j, _ptr(negs), _ptr(fpos), _ptr(lse), _ptr(ids),
                                        _ptr(rows), C.byref(nu), _ptr(rids), _ptr(rrows), C.byref(nr), C.byref(loss)))
        self.synchronize()
        u, r = nu.value, nr.value
        return {"loss": loss.value, "fpos": fpos.cpu().numpy(), "lse": lse.cpu().numpy().reshape(2, nb),
                "node_ids": ids[:u].cpu().numpy().view(np.uint32), "node_rows": rows[:u].cpu().numpy(),
                "rel_ids": rids[:r].cpu().numpy().view(np.uint32), "rel_rows": rrows[:r].cpu().numpy()}

    def adagrad_apply(self, ids, rows, i=0, j=0, relations=False):
        self._enter(ids, rows)
        check(lib().ember_adagrad_apply(self.ctx, _ptr(ids), _ptr(rows), int(ids.numel()), i, j, 1 if relations else 0))
        self._leave()

    def gather(self, ids, i=0, j=0, relations=False, with_acc=True):
        """ParameterSlice gather: (theta, acc) rows of `ids` (device u32), one per
        id in order; node ids must lie in partition i or j (ConfigError otherwise)."""
        t = self.torch
        n = int(ids.numel())
        th = t.empty((n, self.h.dim), dtype=t.float32, device=self.dev)
        ac = t.empty_like(th) if with_acc else None
        self._enter(ids, th, ac)
        check(lib().ember_gather(self.ctx, _ptr(ids), n, i, j, 1 if relations else 0, _ptr(th),
                                 _ptr(ac) if ac is not None else None))
        self._leave()
        return th, ac

    def debug_scores(self, edges, negs, side=0, rows=None, i=0, j=0):
        t = self.torch
        rows = int(edges.shape[0]) if rows is None else rows
        out = t.empty((rows, self.h.num_negatives), dtype=t.float32, device=self.dev)
        self._enter(edges, negs, out)
        check(lib().ember_debug_scores(self.ctx, _ptr(edges), int(edges.shape[0]), i, j, _ptr(negs), side, rows,
                                       _ptr(out)))
        self.synchronize()
        return out.cpu().numpy()

    def debug_sort_slots(self, keys, bits):
        """The step's (key, slot) sort + runs on device keys (uint32 as int32): dict of numpy arrays."""
        t = self.torch
        n = int(keys.numel())
        i32 = dict(dtype=t.int32, device=self.dev)
        out = {k: t.empty(n, **i32) for k in ("keys_sorted", "vals_sorted", "rank", "ukeys")}
        out["uniq"] = t.empty(n, dtype=t.uint8, device=self.dev)
        out["offsets"] = t.empty(n + 1, **i32)
        out["nruns"] = t.empty(1, **i32)
        self._enter(keys, *out.values())
        check(lib().ember_debug_sort_slots(self.ctx, _ptr(keys), n, int(bits), *(_ptr(out[k]) for k in (
            "keys_sorted", "vals_sorted", "rank", "uniq", "ukeys", "offsets", "nruns"))))
        self.synchronize()
        res = {k: v.cpu().numpy() for k, v in out.items()}
        for k in ("keys_sorted", "vals_sorted", "rank", "ukeys", "offsets", "nruns"):
            res[k] = res[k].view(np.uint32)
        return res

    def eval_ranks(self, test_edges, train_edges, n_eval=1000, alpha_eval=0.5, block=1000, eval_seed=7):
        t = self.torch
        n = int(test_edges.shape[0])
        ranks = t.empty(2 * n, dtype=t.int32, device=self.dev)
        self._enter(test_edges, train_edges, ranks)
        check(lib().ember_eval_ranks(self.ctx, _ptr(test_edges), n, _ptr(train_edges), int(train_edges.shape[0]),
                                     n_eval, alpha_eval, block, eval_seed, _ptr(ranks)))
        self.synchronize()
        return ranks.cpu().numpy().view(np.uint32)

    def eval_ranks_filtered(self, test_edges, filter_keys):
        """Filtered ranks against every node; filter_keys: sorted packed u64
        keys (s<<40 | r<<24 | t) of the known triples, on the device (int64 tensor)."""
        t = self.torch
        n = int(test_edges.shape[0])
        ranks = t.empty(2 * n, dtype=t.int32, device=self.dev)
        self._enter(test_edges, filter_keys, ranks)
        check(lib().ember_eval_ranks_filtered(self.ctx, _ptr(test_edges), n, _ptr(filter_keys),
                                              int(filter_keys.numel()), _ptr(ranks)))
        self.synchronize()
        return ranks.cpu().numpy().view(np.uint32)

    def overflow_rows(self) -> int:
        """Rows recomputed exactly because their log-sum-exp left the tensor-core engine's range."""
        v = C.c_uint64(0)
        check(lib().ember_overflow_rows(self.ctx, C.byref(v)))
        return v.value

    def profile(self, enable: bool = True):
        check(lib().ember_profile_enable(self.ctx, 1 if enable else 0))

    def profile_read(self) -> dict:
        ms = (C.c_double * 6)()
        la, lc = C.c_uint64(0), C.c_uint64(0)
        check(lib().ember_profile_read(self.ctx, ms, C.byref(la), C.byref(lc)))
        names = ["sample", "gather", "contraction", "chain_loss", "reduce_adagrad"]
        return {"ms": {n: ms[k] for k, n in enumerate(names)}, "launches": la.value, "lib_calls": lc.value}

    def comm_init(self, unique_id: bytes, rank: int, world: int):
        buf = C.create_string_buffer(unique_id, 128)
        check(lib().ember_comm_init(self.ctx, buf, rank, world))


class PartitionBuffer:
    """PartitionBuffer on the device: `capacity` HBM slots (+2 staging) over a
    pinned-host backing store holding every partition's theta and acc. Replays the plan's bucket
    sequence with Belady eviction, prefetch and asynchronous writeback (csrc/buffer.cu).

    The trainer must be created with allocate=False: the buffer binds its partition tables."""

    def __init__(self, trainer: Trainer, capacity: int, plan_seq, host_theta=None, host_acc=None):
        t = trainer.torch
        self.tr, self.c = trainer, capacity
        p, d = trainer.p, trainer.h.dim
        self.seq = np.ascontiguousarray(np.asarray(plan_seq, dtype=np.uint32).reshape(-1))
        if host_theta is None:
            host_theta = [t.empty((partition_size(trainer.V, p, k), d), dtype=t.float32).pin_memory() for k in range(p)]
            host_acc = [t.empty((partition_size(trainer.V, p, k), d), dtype=t.float32).pin_memory() for k in range(p)]
        self.host_theta, self.host_acc = host_theta, host_acc
        th = (C.c_void_p * p)(*[_ptr(x) for x in host_theta])
        ac = (C.c_void_p * p)(*[_ptr(x) for x in host_acc])
        buf = C.c_void_p()
        check(lib().ember_buffer_create(trainer.ctx, capacity, _ptr(self.seq), len(self.seq) // 2, th, ac,
                                        C.byref(buf)))
        self.buf = buf

    def init_backing(self, seed: int):
        """init_embeddings of every partition, computed on the device and stored to
        the host backing store (bit-identical to a resident init)."""
        t, tr = self.tr.torch, self.tr
        rows = max(x.shape[0] for x in self.host_theta)
        th = t.empty((rows, tr.h.dim), dtype=t.float32, device=tr.dev)
        ac = t.empty((rows, tr.h.dim), dtype=t.float32, device=tr.dev)
        for k in range(tr.p):
            check(lib().ember_tables_bind(tr.ctx, k, _ptr(th), _ptr(ac)))
            check(lib().ember_init_partition(tr.ctx, k, seed))
            tr.torch_stream().synchronize()
            n = self.host_theta[k].shape[0]
            self.host_theta[k].copy_(th[:n])
            self.host_acc[k].copy_(ac[:n])
        if tr.rel_theta is not None:
            check(lib().ember_init_relations(tr.ctx, seed))
        tr.torch_stream().synchronize()

    def train_epoch(self, edges_dev, offsets, epoch: int) -> dict:
        """train_epoch_partitioned through the buffer."""
        st = StepStats()
        off = np.ascontiguousarray(np.asarray(offsets, dtype=np.uint64))
        check(lib().ember_train_epoch_buffered(self.tr.ctx, self.buf, _ptr(edges_dev), _ptr(off), epoch, C.byref(st)))
        return {"loss": st.loss_sum / max(1, st.batches), "batches": st.batches, "edges": st.edges}

    def acquire(self, step: int) -> tuple[int, int]:
        i, j = C.c_uint32(0), C.c_uint32(0)
        check(lib().ember_buffer_acquire(self.buf, step, C.byref(i), C.byref(j)))
        return i.value, j.value

    def release(self, step: int):
        check(lib().ember_buffer_release(self.buf, step))

    def flush(self):
        check(lib().ember_buffer_flush(self.buf))

    def stats(self) -> dict:
        r = BufferReport()
        check(lib().ember_buffer_stats(self.buf, C.byref(r)))
        return {f: getattr(r, f) for f, _ in BufferReport._fields_}

    def decisions(self) -> np.ndarray:
        n = C.c_uint32(0)
        check(lib().ember_buffer_decisions(self.buf, None, C.byref(n)))
        out = np.zeros(3 * max(1, n.value), dtype=np.uint32)
        check(lib().ember_buffer_decisions(self.buf, _ptr(out), C.byref(n)))
        return out[:3 * n.value].reshape(-1, 3)

    def node_table(self):
        """Concatenated host backing store (after flush), in on-disk coordinate order."""
        self.flush()
        k = self.tr.h.kind
        return (rows_to_disk(np.concatenate([x.numpy() for x in self.host_theta]), k),
                rows_to_disk(np.concatenate([x.numpy() for x in self.host_acc]), k))

    def close(self):
        if getattr(self, "buf", None):
            check(lib().ember_buffer_destroy(self.buf))
            self.buf = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
