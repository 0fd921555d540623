"""ctypes binding of libember_b200.so (the C-ABI in include/ember_gpu.h).

The product path is the native library; this module only loads it and declares signatures.
There is no Python or CPU fallback: if the library is missing, import of the op fails loudly.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
# EMBER_LIB: load another build of the same library (A/B timing of two builds in one process tree)
LIB_PATH = os.environ.get("EMBER_LIB") or os.path.join(HERE, "libember_b200.so")

EMBER_OK, EMBER_EUSER, EMBER_EINTERNAL = 0, 1, 2
KIND = {"dot": 0, "distmult": 1, "complex": 2}
ENGINE = {"simt": 0, "tc": 1}
ORDERING = {"elimination": 0, "beta": 0, "hilbert": 1, "hilbert_symmetric": 2, "random": 3}


class ModelDesc(C.Structure):
    _fields_ = [("kind", C.c_int32), ("dim", C.c_uint32), ("lr", C.c_float), ("eps", C.c_float),
                ("batch_size", C.c_uint32), ("num_negatives", C.c_uint32), ("alpha", C.c_float),
                ("num_chunks", C.c_uint32), ("neg_seed", C.c_uint64), ("engine", C.c_int32),
                ("reserved", C.c_uint32)]


class GraphDesc(C.Structure):
    _fields_ = [("num_nodes", C.c_uint64), ("num_relations", C.c_uint32), ("num_partitions", C.c_uint32)]


class StepStats(C.Structure):
    _fields_ = [("loss_sum", C.c_double), ("batches", C.c_uint64), ("edges", C.c_uint64),
                ("unique_nodes", C.c_uint64), ("unique_rels", C.c_uint64)]


class BufferReport(C.Structure):
    _fields_ = [("reads", C.c_uint64), ("writes", C.c_uint64), ("bytes_read", C.c_uint64),
                ("bytes_written", C.c_uint64), ("swaps_per_epoch", C.c_uint64), ("epochs", C.c_uint64),
                ("stalls", C.c_uint32), ("slots", C.c_uint32), ("stall_ms", C.c_double), ("slot_bytes", C.c_uint64)]


class EmberError(RuntimeError):
    pass


class ConfigError(EmberError):
    pass


_LIB = None
vp, u32, u64, f32, i32 = C.c_void_p, C.c_uint32, C.c_uint64, C.c_float, C.c_int


def _declare(L):
    sig = {
        "ember_last_error": (C.c_char_p, []),
        "ember_version": (C.c_int, []),
        "ember_ctx_create": (C.c_int, [i32, C.POINTER(ModelDesc), C.POINTER(GraphDesc), vp, C.POINTER(vp)]),
        "ember_ctx_destroy": (C.c_int, [vp]),
        "ember_ctx_stream": (vp, [vp]),
        "ember_ctx_synchronize": (C.c_int, [vp]),
        "ember_tables_bind": (C.c_int, [vp, u32, vp, vp]),
        "ember_relations_bind": (C.c_int, [vp, vp, vp]),
        "ember_init_partition": (C.c_int, [vp, u32, u64]),
        "ember_init_relations": (C.c_int, [vp, u64]),
        "ember_train_batch": (C.c_int, [vp, vp, u64, u64, u32, u32, u32, u64, u32, u32, vp]),
        "ember_train_bucket": (C.c_int, [vp, vp, u64, u32, u32, u64, u32, C.POINTER(StepStats)]),
        "ember_train_epoch": (C.c_int, [vp, vp, vp, vp, u64, C.POINTER(StepStats)]),
        "ember_train_batch_host": (C.c_int, [vp, vp, u64, vp, u32, u32, u32, u64, u32, u32, vp]),
        "ember_sample_negatives": (C.c_int, [vp, vp, u64, u32, u32, u64, u32, u32, vp]),
        "ember_loss_and_grad": (C.c_int, [vp, vp, u32, u32, u32, vp, vp, vp, vp, vp, C.POINTER(u32), vp, vp,
                                          C.POINTER(u32), C.POINTER(C.c_double)]),
        "ember_adagrad_apply": (C.c_int, [vp, vp, vp, u32, u32, u32, i32]),
        "ember_gather": (C.c_int, [vp, vp, u32, u32, u32, i32, vp, vp]),
        "ember_debug_scores": (C.c_int, [vp, vp, u32, u32, u32, vp, i32, u32, vp]),
        "ember_debug_sort_slots": (C.c_int, [vp, vp, u32, u32, vp, vp, vp, vp, vp, vp, vp]),
        "ember_eval_ranks": (C.c_int, [vp, vp, u32, vp, u64, u32, f32, u32, u64, vp]),
        "ember_eval_ranks_filtered": (C.c_int, [vp, vp, u32, vp, u64, vp]),
        "ember_make_plan": (C.c_int, [i32, u32, u32, u64, vp, C.POINTER(u64), vp, C.POINTER(u32), vp, vp]),
        "ember_lower_bound_swaps": (u64, [u32, u32]),
        "ember_elimination_swap_formula": (u64, [u32, u32]),
        "ember_graph_generate": (C.c_int, [i32, u64, u32, u64, u64, f32, f32, vp, vp]),
        "ember_graph_bucket": (C.c_int, [i32, u64, u32, vp, u64, vp, vp]),
        "ember_graph_preprocess": (C.c_int, [i32, vp, u64, u32, u64, f32, f32, vp, vp, vp, vp, vp, vp, vp,
                                             C.POINTER(u64), C.POINTER(u32)]),
        "ember_tc_selftest": (C.c_int, [i32, i32, i32, i32, u64, C.POINTER(C.c_double)]),
        "ember_tc_mmabench": (C.c_int, [i32, i32, i32, i32, C.POINTER(C.c_double)]),
        "ember_profile_enable": (C.c_int, [vp, i32]),
        "ember_profile_read": (C.c_int, [vp, vp, C.POINTER(u64), C.POINTER(u64)]),
        "ember_buffer_create": (C.c_int, [vp, u32, vp, u32, vp, vp, C.POINTER(vp)]),
        "ember_buffer_destroy": (C.c_int, [vp]),
        "ember_buffer_acquire": (C.c_int, [vp, u32, C.POINTER(u32), C.POINTER(u32)]),
        "ember_buffer_release": (C.c_int, [vp, u32]),
        "ember_buffer_flush": (C.c_int, [vp]),
        "ember_buffer_stats": (C.c_int, [vp, C.POINTER(BufferReport)]),
        "ember_buffer_decisions": (C.c_int, [vp, vp, C.POINTER(u32)]),
        "ember_train_epoch_buffered": (C.c_int, [vp, vp, vp, vp, u64, C.POINTER(StepStats)]),
        "ember_make_rounds": (C.c_int, [u32, u32, vp, vp, vp, vp, C.POINTER(u32)]),
        "ember_make_rounds_overlap": (C.c_int, [u32, u32, vp, vp, vp, vp, vp, C.POINTER(u32)]),
        "ember_dist_plan": (C.c_int, [u32, u32, u32, C.c_int, vp, u32, vp, vp, C.POINTER(u64)]),
        "ember_dist_run": (C.c_int, [u32, u32, u32, C.c_int, vp, u32, u64, u64, u64, vp, vp]),
        "ember_dist_create": (C.c_int, [vp, u32, u32, C.c_int, vp, vp, vp, vp, C.POINTER(vp)]),
        "ember_dist_destroy": (C.c_int, [vp]),
        "ember_dist_init_embeddings": (C.c_int, [vp, u64]),
        "ember_dist_train_epoch": (C.c_int, [vp, u64, u64, u64, vp]),
        "ember_dist_tables": (C.c_int, [vp, u32, C.POINTER(vp), C.POINTER(vp)]),
        "ember_dist_synchronize": (C.c_int, [vp]),
        "ember_dist_loss": (C.c_int, [vp, vp]),
        "ember_nccl_unique_id": (C.c_int, [vp]),
        "ember_relations_external": (C.c_int, [vp, vp]),
        "ember_relations_apply_dense": (C.c_int, [vp, vp]),
        "ember_overflow_rows": (C.c_int, [vp, C.POINTER(u64)]),
        "ember_device_alloc": (C.c_int, [vp, C.c_size_t, C.POINTER(vp)]),
        "ember_device_free": (C.c_int, [vp, vp]),
        "ember_copy_to_device": (C.c_int, [vp, vp, vp, C.c_size_t]),
        "ember_copy_to_host": (C.c_int, [vp, vp, vp, C.c_size_t]),
        "ember_host_alloc_pinned": (C.c_int, [C.c_size_t, C.POINTER(vp)]),
        "ember_host_free_pinned": (C.c_int, [vp]),
        "ember_tables_allocate": (C.c_int, [vp, u32]),
        "ember_tables_get": (C.c_int, [vp, u32, C.POINTER(vp), C.POINTER(vp), C.POINTER(u64)]),
        "ember_rows_layout": (C.c_int, [vp, vp, u64, C.c_int]),
        "ember_rows_layout_host": (C.c_int, [C.c_int, u32, vp, u64, C.c_int]),
        "ember_comm_init": (C.c_int, [vp, vp, i32, i32]),
        "ember_comm_barrier": (C.c_int, [vp]),
        "ember_partition_copy": (C.c_int, [vp, vp, vp, i32, vp, vp, i32, u64]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(L, name)
        fn.restype = res
        fn.argtypes = args
    return L


EXPORTED = None  # filled on load: the symbol names declared above


def lib():
    """Loads the native library; raises if it has not been built (no fallback)."""
    global _LIB
    if _LIB is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} missing: build it with `python -c 'import __graft_entry__ as g; g.build()'`"
                              " (make -C paper_2101_08358_b200/csrc)")
        _LIB = _declare(C.CDLL(LIB_PATH))
    return _LIB


def check(status: int) -> None:
    if status == EMBER_OK:
        return
    msg = lib().ember_last_error().decode(errors="replace")
    if status == EMBER_EUSER:
        raise ConfigError(msg)
    raise EmberError(msg)
