"""Shared setup for the -m gpu parity tests: a small partitioned synthetic graph with identical
initial parameters on the device (product) and on the host (oracle)."""
import numpy as np

import paper_2101_08358_b200 as eb
from oracle import pyoracle as po


def make_graph(V=3000, R=20, E=20000, p=1, seed=5):
    edges, split = eb.generate_graph(V, R, E, seed=seed, train_frac=0.9, valid_frac=0.05)
    train = edges[split == 0]
    bucketed, offsets = eb.bucket_edges(train, V, p)
    return bucketed, offsets, edges[split == 2]


def make_trainer(kind="distmult", dim=32, b=512, nt=64, alpha=0.5, chunks=1, V=3000, R=20, p=1, engine="simt",
                 init_seed=11, neg_seed=3):
    h = eb.Hyper(kind=kind, dim=dim, batch_size=b, num_negatives=nt, alpha=alpha, num_chunks=chunks,
                 neg_seed=neg_seed, engine=engine)
    tr = eb.Trainer(h, V, R, p, device=0)
    tr.init_embeddings(init_seed)
    tr.synchronize()
    return tr


def host_tables(tr):
    th, ac = tr.node_table()
    if tr.rel_theta is not None:
        rt, ra = tr.relation_table()
    else:
        rt = np.zeros((1, tr.h.dim), np.float32)
        ra = np.zeros((1, tr.h.dim), np.float32)
    return th.copy(), ac.copy(), rt, ra


def oracle_model(tr):
    h = tr.h
    return po.model(h.kind, dim=h.dim, lr=h.lr, eps=h.eps, n_t=h.num_negatives, alpha=h.alpha, chunks=h.num_chunks,
                    seed=h.neg_seed)


def rel_err(a, b):
    """max |a - b| / max |b| over the whole tensor."""
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-30)) if b.size else 0.0


def row_rel_err(a, b, floor=1e-3):
    """max over rows of ||a_r - b_r|| / max(||b_r||, floor * max_r ||b_r||)."""
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    if b.size == 0:
        return 0.0
    nb = np.linalg.norm(b, axis=1)
    den = np.maximum(nb, floor * nb.max())
    return float((np.linalg.norm(a - b, axis=1) / den).max())
