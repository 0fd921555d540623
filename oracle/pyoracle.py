"""ctypes bindings for the CPU oracle (liboracle.so) and the reference build (_ref/libember_ref.so).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference legs. The product package never imports this module.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
_ORACLE = None
_REF = None

u32p = np.ctypeslib.ndpointer(np.uint32, flags="C_CONTIGUOUS")
u64p = np.ctypeslib.ndpointer(np.uint64, flags="C_CONTIGUOUS")
f32p = np.ctypeslib.ndpointer(np.float32, flags="C_CONTIGUOUS")
f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")

KINDS = {"dot": 0, "distmult": 1, "complex": 2}


class OrcModel(C.Structure):
    _fields_ = [
        ("kind", C.c_int32),
        ("dim", C.c_uint32),
        ("lr", C.c_float),
        ("eps", C.c_float),
        ("num_negatives", C.c_uint32),
        ("alpha", C.c_float),
        ("num_chunks", C.c_uint32),
        ("pad_", C.c_uint32),
        ("neg_seed", C.c_uint64),
    ]


def build(ref: bool = False) -> None:
    subprocess.run(["make", "-s", "-C", HERE, "all"], check=True)
    if ref and os.path.isdir("/root/reference/proj"):
        subprocess.run(["make", "-s", "-C", HERE, "ref"], check=True)


def lib():
    global _ORACLE
    if _ORACLE is None:
        path = os.path.join(HERE, "liboracle.so")
        if not os.path.exists(path):
            build()
        L = C.CDLL(path)
        L.orc_splitmix64.restype = C.c_uint64
        L.orc_splitmix64.argtypes = [C.c_uint64]
        L.orc_mix_seed.restype = C.c_uint64
        L.orc_mix_seed.argtypes = [C.c_uint64, C.c_uint64]
        L.orc_mix_seed3.restype = C.c_uint64
        L.orc_mix_seed3.argtypes = [C.c_uint64, C.c_uint64, C.c_uint64]
        L.orc_rng_next.argtypes = [C.c_uint64, C.c_uint32, u64p]
        L.orc_rng_uniform_below.argtypes = [C.c_uint64, C.c_uint64, C.c_uint32, u64p]
        L.orc_rng_uniform.argtypes = [C.c_uint64, C.c_float, C.c_float, C.c_uint32, f32p]
        L.orc_part_offset.restype = C.c_uint64
        L.orc_part_offset.argtypes = [C.c_uint64, C.c_uint32, C.c_uint32]
        L.orc_part_size.restype = C.c_uint64
        L.orc_part_size.argtypes = [C.c_uint64, C.c_uint32, C.c_uint32]
        L.orc_score.restype = C.c_float
        L.orc_score.argtypes = [C.c_int32, C.c_uint32, f32p, f32p, f32p]
        L.orc_init_rows.argtypes = [C.c_uint64, C.c_uint32, C.c_uint64, C.c_uint64, f32p]
        L.orc_sample_negatives.argtypes = [C.POINTER(OrcModel), C.c_uint64, C.c_uint32, C.c_uint32, u32p, C.c_uint64,
                                           C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint64, u32p]
        L.orc_loss_and_grad.restype = C.c_double
        L.orc_loss_and_grad.argtypes = [C.POINTER(OrcModel), u32p, C.c_uint32, u32p, f32p, f32p, f32p, f32p, u32p,
                                        f32p, C.POINTER(C.c_uint32), u32p, f32p, C.POINTER(C.c_uint32)]
        L.orc_adagrad_apply.argtypes = [C.c_uint32, C.c_float, C.c_float, u32p, f32p, C.c_uint32, f32p, f32p]
        L.orc_train_batch.restype = C.c_double
        L.orc_train_batch.argtypes = [C.POINTER(OrcModel), C.c_uint64, C.c_uint32, C.c_uint32, u32p, C.c_uint64,
                                      C.c_uint64, C.c_uint32, C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint64, f32p,
                                      f32p, f32p, f32p]
        L.orc_eval_ranks.argtypes = [C.c_int32, C.c_uint32, f32p, f32p, C.c_uint64, u32p, C.c_uint32, C.c_int,
                                     u64p, C.c_uint64, u32p, C.c_uint64, C.c_uint32, C.c_float, C.c_uint32,
                                     C.c_uint64, u32p]
        L.orc_aggregate.argtypes = [u32p, C.c_uint64, u32p, C.c_uint32, f64p]
        L.orc_preprocess.argtypes = [u32p, C.c_uint64, C.c_uint32, C.c_uint64, C.c_float, C.c_float, u32p, u64p, u32p,
                                     u32p, u64p, u32p, u32p, C.POINTER(C.c_uint64), C.POINTER(C.c_uint32)]
        u8p = np.ctypeslib.ndpointer(np.uint8, flags="C_CONTIGUOUS")
        L.orc_graph_generate.argtypes = [C.c_uint64, C.c_uint32, C.c_uint64, C.c_uint64, C.c_uint64, C.c_float,
                                         C.c_float, u32p, u8p]
        L.orc_graph_bucket.restype = C.c_uint64
        L.orc_graph_bucket.argtypes = [C.c_uint64, C.c_uint32, u32p, C.c_void_p, C.c_uint8, C.c_uint64, u32p, u64p]
        L.orc_train_batch_parts.restype = C.c_double
        L.orc_train_batch_parts.argtypes = [C.POINTER(OrcModel), C.c_uint64, C.c_uint32, C.c_uint32, C.c_void_p,
                                            C.c_uint64, C.c_uint64, C.c_uint32, C.c_uint64, C.c_uint64, C.c_void_p,
                                            C.c_void_p, C.c_uint64, C.c_uint64, C.c_void_p, C.c_void_p, C.c_void_p,
                                            C.c_void_p, C.POINTER(C.c_uint32)]
        L.orc_num_threads.restype = C.c_int
        L.orc_set_num_threads.argtypes = [C.c_int]
        _ORACLE = L
    return _ORACLE


def ref_lib():
    """The reference's own ordering.cpp + common.h, compiled by oracle/Makefile into _ref/."""
    global _REF
    if _REF is None:
        path = os.path.join(HERE, "_ref", "libember_ref.so")
        if not os.path.exists(path):
            build(ref=True)
        if not os.path.exists(path):
            return None
        L = C.CDLL(path)
        L.ref_make_plan.argtypes = [C.c_int, C.c_uint32, C.c_uint32, C.c_uint64, u32p, C.POINTER(C.c_uint64), u32p,
                                    C.POINTER(C.c_uint32), u32p, u32p]
        L.ref_lower_bound_swaps.restype = C.c_uint64
        L.ref_lower_bound_swaps.argtypes = [C.c_uint32, C.c_uint32]
        L.ref_elimination_swap_formula.restype = C.c_uint64
        L.ref_elimination_swap_formula.argtypes = [C.c_uint32, C.c_uint32]
        L.ref_simulate_io.argtypes = [C.c_int, C.c_uint32, C.c_uint32, C.c_uint64, C.c_uint64, u64p]
        L.ref_hilbert_d2xy.argtypes = [C.c_uint32, C.c_uint64, u32p]
        L.ref_splitmix64.restype = C.c_uint64
        L.ref_splitmix64.argtypes = [C.c_uint64]
        L.ref_mix_seed.restype = C.c_uint64
        L.ref_mix_seed.argtypes = [C.c_uint64, C.c_uint64]
        L.ref_mix_seed3.restype = C.c_uint64
        L.ref_mix_seed3.argtypes = [C.c_uint64, C.c_uint64, C.c_uint64]
        L.ref_rng_next.argtypes = [C.c_uint64, C.c_uint32, u64p]
        L.ref_rng_uniform_below.argtypes = [C.c_uint64, C.c_uint64, C.c_uint32, u64p]
        L.ref_rng_uniform.argtypes = [C.c_uint64, C.c_float, C.c_float, C.c_uint32, f32p]
        L.ref_rng_shuffle_iota.argtypes = [C.c_uint64, C.c_uint32, u32p]
        _REF = L
    return _REF


def ref_plan(kind: int, p: int, c: int, seed: int):
    """Reference make_plan (ordering.cpp:384) -> dict of numpy arrays, or raises on ConfigError."""
    L = ref_lib()
    seq = np.zeros(2 * p * p, np.uint32)
    adm = np.zeros(c + 2 * p * p + 1, np.uint32)
    swaps = np.zeros(6 * p * p + 3, np.uint32)
    state = np.zeros(p * p, np.uint32)
    sc = C.c_uint64(0)
    na = C.c_uint32(0)
    st = L.ref_make_plan(kind, p, c, seed, seq, C.byref(sc), adm, C.byref(na), swaps, state)
    if st != 0:
        raise ValueError(f"reference make_plan status {st}")
    n = int(sc.value)
    return {"seq": seq.reshape(-1, 2), "swap_count": n, "admissions": adm[: na.value].copy(),
            "swaps": swaps[: 3 * n].reshape(-1, 3).copy(), "bucket_state": state}


def model(kind="distmult", dim=8, lr=0.1, eps=1e-10, n_t=4, alpha=0.5, chunks=1, seed=1) -> OrcModel:
    return OrcModel(KINDS[kind] if isinstance(kind, str) else int(kind), dim, lr, eps, n_t, alpha, chunks, 0, seed)


def part_offset(V, p, k):
    return int(lib().orc_part_offset(V, p, k))


def part_size(V, p, k):
    return int(lib().orc_part_size(V, p, k))


def init_rows(seed, dim, row_begin, rows):
    out = np.zeros(rows * dim, np.float32)
    lib().orc_init_rows(seed, dim, row_begin, rows, out)
    return out.reshape(rows, dim)


def sample_negatives(m: OrcModel, epoch, bucket_step, batch_in_bucket, bucket_edges, src_off, src_size, dst_off,
                     dst_size):
    be = np.ascontiguousarray(bucket_edges, np.uint32).reshape(-1)
    out = np.zeros(max(1, m.num_chunks) * 2 * m.num_negatives, np.uint32)
    lib().orc_sample_negatives(C.byref(m), epoch, bucket_step, batch_in_bucket, be if be.size else np.zeros(3, np.uint32),
                               be.size // 3, src_off, src_size, dst_off, dst_size, out)
    return out


def loss_and_grad(m: OrcModel, edges, negs, node_theta, rel_theta):
    edges = np.ascontiguousarray(edges, np.uint32).reshape(-1)
    nb = edges.size // 3
    d = m.dim
    nneg = negs.size
    cap = 2 * nb + nneg
    fpos = np.zeros(nb, np.float32)
    lse = np.zeros(2 * nb, np.float32)
    ids = np.zeros(cap, np.uint32)
    rows = np.zeros(cap * d, np.float32)
    rids = np.zeros(max(nb, 1), np.uint32)
    rrows = np.zeros(max(nb, 1) * d, np.float32)
    nu = C.c_uint32(0)
    nr = C.c_uint32(0)
    rt = np.ascontiguousarray(rel_theta, np.float32).reshape(-1)
    if rt.size == 0:
        rt = np.zeros(d, np.float32)
    loss = lib().orc_loss_and_grad(C.byref(m), edges, nb, np.ascontiguousarray(negs, np.uint32),
                                   np.ascontiguousarray(node_theta, np.float32).reshape(-1), rt, fpos, lse, ids, rows,
                                   C.byref(nu), rids, rrows, C.byref(nr))
    u, r = nu.value, nr.value
    return {"loss": loss, "fpos": fpos, "lse": lse.reshape(2, nb), "node_ids": ids[:u].copy(),
            "node_rows": rows[: u * d].reshape(u, d).copy(), "rel_ids": rids[:r].copy(),
            "rel_rows": rrows[: r * d].reshape(r, d).copy()}


def adagrad_apply(dim, lr, eps, ids, rows, theta, acc):
    lib().orc_adagrad_apply(dim, lr, eps, np.ascontiguousarray(ids, np.uint32),
                            np.ascontiguousarray(rows, np.float32).reshape(-1), len(ids), theta.reshape(-1),
                            acc.reshape(-1))


def train_batch(m: OrcModel, epoch, bucket_step, batch_in_bucket, bucket_edges, batch_begin, nb, src_off, src_size,
                dst_off, dst_size, node_theta, node_acc, rel_theta, rel_acc):
    be = np.ascontiguousarray(bucket_edges, np.uint32).reshape(-1)
    return lib().orc_train_batch(C.byref(m), epoch, bucket_step, batch_in_bucket, be, be.size // 3, batch_begin, nb,
                                 src_off, src_size, dst_off, dst_size, node_theta.reshape(-1), node_acc.reshape(-1),
                                 rel_theta.reshape(-1), rel_acc.reshape(-1))


def pack_keys(edges):
    e = np.asarray(edges, np.uint64).reshape(-1, 3)
    return np.unique((e[:, 0] << np.uint64(40)) | (e[:, 1] << np.uint64(24)) | e[:, 2])


def eval_ranks(kind, dim, node_theta, rel_theta, num_nodes, test_edges, filtered=False, filter_keys=None,
               train_edges=None, n_eval_neg=1000, alpha_eval=0.5, block=1000, eval_seed=7):
    test = np.ascontiguousarray(test_edges, np.uint32).reshape(-1)
    n = test.size // 3
    ranks = np.zeros(2 * n, np.uint32)
    fk = np.ascontiguousarray(filter_keys if filter_keys is not None else np.zeros(1, np.uint64), np.uint64)
    tr = np.ascontiguousarray(train_edges if train_edges is not None else np.zeros(3, np.uint32), np.uint32).reshape(-1)
    rt = np.ascontiguousarray(rel_theta, np.float32).reshape(-1)
    if rt.size == 0:
        rt = np.zeros(dim, np.float32)
    lib().orc_eval_ranks(KINDS[kind] if isinstance(kind, str) else int(kind), dim,
                         np.ascontiguousarray(node_theta, np.float32).reshape(-1), rt, num_nodes, test, n,
                         1 if filtered else 0, fk, fk.size if filter_keys is not None else 0, tr, tr.size // 3,
                         n_eval_neg, alpha_eval, block, eval_seed, ranks)
    return ranks


def aggregate(ranks, ks=(1, 10)):
    ks_a = np.asarray(ks, np.uint32)
    out = np.zeros(1 + len(ks), np.float64)
    lib().orc_aggregate(np.ascontiguousarray(ranks, np.uint32), len(ranks), ks_a, len(ks), out)
    return {"mrr": out[0], **{f"hits@{k}": out[1 + i] for i, k in enumerate(ks)}}


def preprocess(raw, p, seed, train_frac=0.9, valid_frac=0.05):
    """orc_preprocess (graph-store preprocessing restated on the CPU): same outputs as
    paper_2101_08358_b200.preprocess_graph, as numpy arrays."""
    raw = np.ascontiguousarray(raw, np.uint32).reshape(-1, 3)
    n = raw.shape[0]
    train = np.zeros((n, 3), np.uint32)
    valid = np.zeros((n, 3), np.uint32)
    test = np.zeros((n, 3), np.uint32)
    off = np.zeros(p * p + 1, np.uint64)
    counts = np.zeros(3, np.uint64)
    ntok = np.zeros(2 * n, np.uint32)
    rtok = np.zeros(n, np.uint32)
    V, R = C.c_uint64(0), C.c_uint32(0)
    lib().orc_preprocess(raw, n, p, seed, C.c_float(train_frac), C.c_float(valid_frac), train, off, valid, test,
                         counts, ntok, rtok, C.byref(V), C.byref(R))
    a, b, c = (int(x) for x in counts)
    return {"train": train[:a], "valid": valid[:b], "test": test[:c], "offsets": off, "num_nodes": V.value,
            "num_relations": R.value, "node_tokens": ntok[:V.value], "rel_tokens": rtok[:R.value]}


def graph_generate(V, R, n, seed, train_frac=0.9, valid_frac=0.05, first=0):
    """The benchmark graph generator restated on the CPU (orc_graph_generate): (edges (n,3) u32, split (n,) u8)."""
    edges = np.zeros((n, 3), np.uint32)
    split = np.zeros(n, np.uint8)
    lib().orc_graph_generate(V, R, first, n, seed, C.c_float(train_frac), C.c_float(valid_frac),
                             edges.reshape(-1), split)
    return edges, split


def graph_bucket(V, p, edges, split=None, which=0):
    """bucket_edges of the edges whose split byte == which (split None: all):
    (bucketed (m,3) u32, offsets (p*p+1,) u64)."""
    edges = np.ascontiguousarray(edges, np.uint32).reshape(-1, 3)
    n = edges.shape[0]
    if split is not None:
        split = np.ascontiguousarray(split, np.uint8)
        m = int(np.count_nonzero(split == which))
    else:
        m = n
    out = np.zeros((max(m, 1), 3), np.uint32)
    off = np.zeros(p * p + 1, np.uint64)
    lib().orc_graph_bucket(V, p, edges.reshape(-1), split.ctypes.data if split is not None else None, which, n,
                           out.reshape(-1), off)
    return out[:m], off


def train_batch_parts(m: OrcModel, epoch, bucket_step, batch_in_bucket, bucket_edges, batch_begin, nb, part_i, part_j,
                      rel_theta, rel_acc):
    """The CPU trainer's step on partitions (orc_train_batch_parts): part_* = (first_row, theta, acc) with
    theta/acc (rows, dim) f32 arrays updated in place. Returns (loss, unique node rows)."""
    be = np.ascontiguousarray(bucket_edges, np.uint32)
    fi, ti, ai = part_i
    fj, tj, aj = part_j
    nu = C.c_uint32(0)
    loss = lib().orc_train_batch_parts(C.byref(m), epoch, bucket_step, batch_in_bucket, be.ctypes.data, be.size // 3,
                                       batch_begin, nb, fi, ti.shape[0], ti.ctypes.data, ai.ctypes.data, fj,
                                       tj.shape[0], tj.ctypes.data, aj.ctypes.data, rel_theta.ctypes.data,
                                       rel_acc.ctypes.data, C.byref(nu))
    return loss, nu.value
