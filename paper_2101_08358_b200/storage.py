"""The ember graph store's on-disk files, for checkpoints and the partition
buffer's backing store. Formats follow the reference (proj/include/ember/binary_io.h; C++
restatement in include/ember/binary_io.h): little-endian 32-bit floats, 32-bit ids, 64-bit offsets.

  meta.json              GraphMeta manifest (num_nodes, num_relations, num_partitions, dim, ...)
  edges_<split>.bin      (src, rel, dst) u32 triples, bucketed by (part(src), part(dst))
  bucket_offsets.bin     p*p + 1 u64 offsets into edges_train.bin
  node_part_<k>.bin      rows_k x d f32 parameters, immediately followed by rows_k x d f32 Adagrad state
  relations.bin          |R| x d f32 parameters followed by |R| x d f32 Adagrad state
"""
from __future__ import annotations

import json
import os

import numpy as np

from . import partition_size, rows_to_disk, rows_to_hbm


def _pod_write(path: str, arr: np.ndarray) -> None:
    np.ascontiguousarray(arr).tofile(path)


def _pod_read_exact(path: str, dtype, count: int) -> np.ndarray:
    want = count * np.dtype(dtype).itemsize
    have = os.path.getsize(path)
    if have != want:
        raise OSError(f"file {path} has {have} bytes, expected {want}")  # IoError (binary_io.h)
    return np.fromfile(path, dtype=dtype, count=count)


def write_meta(root: str, num_nodes: int, num_relations: int, num_partitions: int, dim: int, **extra) -> None:
    os.makedirs(root, exist_ok=True)
    meta = {"num_nodes": int(num_nodes), "num_relations": int(num_relations),
            "num_partitions": int(num_partitions), "dim": int(dim), **extra}
    with open(os.path.join(root, "meta.json"), "w") as f:
        json.dump(meta, f, indent=1, sort_keys=True)


def read_meta(root: str) -> dict:
    with open(os.path.join(root, "meta.json")) as f:
        return json.load(f)


def write_edges(root: str, split: str, edges: np.ndarray, bucket_offsets: np.ndarray | None = None) -> None:
    os.makedirs(root, exist_ok=True)
    _pod_write(os.path.join(root, f"edges_{split}.bin"), np.asarray(edges, np.uint32).reshape(-1, 3))
    if bucket_offsets is not None:
        _pod_write(os.path.join(root, "bucket_offsets.bin"), np.asarray(bucket_offsets, np.uint64))


def read_edges(root: str, split: str) -> np.ndarray:
    path = os.path.join(root, f"edges_{split}.bin")
    n = os.path.getsize(path)
    if n % 12:
        raise OSError(f"file size {n} not a multiple of element size: {path}")
    return np.fromfile(path, dtype=np.uint32).reshape(-1, 3)


def read_bucket_offsets(root: str, p: int) -> np.ndarray:
    return _pod_read_exact(os.path.join(root, "bucket_offsets.bin"), np.uint64, p * p + 1)


def write_node_part(root: str, k: int, theta: np.ndarray, acc: np.ndarray) -> None:
    os.makedirs(root, exist_ok=True)
    with open(os.path.join(root, f"node_part_{k}.bin"), "wb") as f:
        np.ascontiguousarray(theta, np.float32).tofile(f)
        np.ascontiguousarray(acc, np.float32).tofile(f)


def read_node_part(root: str, k: int, rows: int, dim: int, out_theta=None, out_acc=None):
    """Partition k's (theta, acc); with out_* (e.g. pinned host tensors as numpy views) the file is
    read straight into them."""
    data = _pod_read_exact(os.path.join(root, f"node_part_{k}.bin"), np.float32, 2 * rows * dim)
    th, ac = data[: rows * dim].reshape(rows, dim), data[rows * dim:].reshape(rows, dim)
    if out_theta is not None:
        out_theta[...] = th
        out_acc[...] = ac
        return out_theta, out_acc
    return th, ac


def write_relations(root: str, theta: np.ndarray, acc: np.ndarray) -> None:
    os.makedirs(root, exist_ok=True)
    with open(os.path.join(root, "relations.bin"), "wb") as f:
        np.ascontiguousarray(theta, np.float32).tofile(f)
        np.ascontiguousarray(acc, np.float32).tofile(f)


def read_relations(root: str, num_relations: int, dim: int):
    data = _pod_read_exact(os.path.join(root, "relations.bin"), np.float32, 2 * num_relations * dim)
    n = num_relations * dim
    return data[:n].reshape(num_relations, dim), data[n:].reshape(num_relations, dim)


def save_trainer(root: str, trainer) -> None:
    """Checkpoint of a Trainer with HBM-resident tables (every partition + relations)."""
    trainer.synchronize()
    write_meta(root, trainer.V, trainer.R, trainer.p, trainer.h.dim, model=trainer.h.kind)
    kind = trainer.h.kind  # the files hold on-disk coordinate order, the tables the HBM layout
    for k in range(trainer.p):
        write_node_part(root, k, rows_to_disk(trainer.theta[k].cpu().numpy(), kind),
                        rows_to_disk(trainer.acc[k].cpu().numpy(), kind))
    if trainer.rel_theta is not None:
        write_relations(root, *trainer.relation_table())


def load_trainer(root: str, trainer) -> None:
    """Restores a checkpoint written by save_trainer into a Trainer of the same geometry."""
    meta = read_meta(root)
    if (meta["num_nodes"], meta["num_relations"], meta["num_partitions"], meta["dim"]) != \
            (trainer.V, trainer.R, trainer.p, trainer.h.dim):
        raise ValueError("checkpoint geometry does not match the trainer")  # ConfigError
    t, kind = trainer.torch, trainer.h.kind
    for k in range(trainer.p):
        th, ac = read_node_part(root, k, partition_size(trainer.V, trainer.p, k), trainer.h.dim)
        trainer.theta[k].copy_(t.from_numpy(rows_to_hbm(th, kind)))
        trainer.acc[k].copy_(t.from_numpy(rows_to_hbm(ac, kind)))
    if trainer.rel_theta is not None:
        th, ac = read_relations(root, trainer.R, trainer.h.dim)
        trainer.rel_theta.copy_(t.from_numpy(rows_to_hbm(th, kind)))
        trainer.rel_acc.copy_(t.from_numpy(rows_to_hbm(ac, kind)))
    trainer.synchronize()


def load_buffer_backing(root: str, buf) -> None:
    """Fills a PartitionBuffer's pinned host backing store from node_part_<k>.bin files."""
    tr = buf.tr  # the backing store holds the HBM row layout
    for k in range(tr.p):
        th, ac = read_node_part(root, k, buf.host_theta[k].shape[0], tr.h.dim)
        buf.host_theta[k].numpy()[:] = rows_to_hbm(th, tr.h.kind)
        buf.host_acc[k].numpy()[:] = rows_to_hbm(ac, tr.h.kind)


def save_buffer_backing(root: str, buf) -> None:
    """Writes the backing store (after an epoch, i.e. after the buffer's flush) as node_part files."""
    buf.flush()
    kind = buf.tr.h.kind
    for k in range(buf.tr.p):
        write_node_part(root, k, rows_to_disk(buf.host_theta[k].numpy(), kind),
                        rows_to_disk(buf.host_acc[k].numpy(), kind))
