"""Test infrastructure: a DistributedTrainer backend over the CPU oracle (oracle/), so the
multi-GPU orchestration (round schedule, lockstep relation all-reduce, partition handoff) runs
with gloo on CPU. Never used by the product path."""
from __future__ import annotations

import contextlib

import numpy as np
import torch

import paper_2101_08358_b200 as eb
from oracle import pyoracle as po


class OracleBackend:
    def __init__(self, kind, dim, V, R, p, nt, alpha, neg_seed, edges, lr=0.1, eps=1e-10):
        self.m = po.model(kind, dim=dim, lr=lr, eps=eps, n_t=nt, alpha=alpha, chunks=1, seed=neg_seed)
        self.kind, self.d, self.V, self.R, self.p = kind, dim, V, R, p
        self.lr, self.eps = lr, eps
        self.edges = edges  # bucketed u32 [n, 3]
        # full-size tables; only the rows of held partitions are meaningful on this rank
        self.theta = np.full((V, dim), np.nan, np.float32)
        self.acc = np.full((V, dim), np.nan, np.float32)
        self.held: set[int] = set()
        self.rel_theta = np.zeros((max(R, 1), dim), np.float32)
        self.rel_acc = np.zeros((max(R, 1), dim), np.float32)
        self.rel_grad_t = torch.zeros((max(R, 1), dim), dtype=torch.float32)

    def _sl(self, x):
        o = eb.partition_offset(self.V, self.p, x)
        return slice(o, o + eb.partition_size(self.V, self.p, x))

    def init_partition(self, x, seed):
        s = self._sl(x)
        self.theta[s] = po.init_rows(seed, self.d, s.start, s.stop - s.start)
        self.acc[s] = 0
        self.held.add(x)

    def init_relations(self, seed):
        if self.kind != "dot":
            self.rel_theta[:] = po.init_rows(seed ^ 0x52454C, self.d, 0, self.R)
            self.rel_acc[:] = 0

    def tables(self, x):
        s = self._sl(x)
        return torch.from_numpy(self.theta[s]), torch.from_numpy(self.acc[s])

    def empty_tables(self, x):
        n = eb.partition_size(self.V, self.p, x)
        return torch.empty((n, self.d)), torch.empty((n, self.d))

    def adopt(self, x, th, ac):
        s = self._sl(x)
        self.theta[s] = th.numpy()
        self.acc[s] = ac.numpy()
        self.held.add(x)

    def drop(self, x):
        self.theta[self._sl(x)] = np.nan
        self.acc[self._sl(x)] = np.nan
        self.held.discard(x)

    def train_batch(self, pos, i, j, k, lo, hi, begin, nb, epoch):
        assert i in self.held and j in self.held, f"bucket ({i},{j}) not resident on this rank"
        bucket = self.edges[lo:hi]
        si, sj = self._sl(i), self._sl(j)
        negs = po.sample_negatives(self.m, epoch, pos, k, bucket, si.start, si.stop - si.start, sj.start,
                                   sj.stop - sj.start)
        g = po.loss_and_grad(self.m, bucket[begin:begin + nb], negs, self.theta, self.rel_theta)
        po.adagrad_apply(self.d, self.lr, self.eps, g["node_ids"], g["node_rows"], self.theta, self.acc)
        self.rel_grad_t.zero_()
        if self.kind != "dot" and len(g["rel_ids"]):
            self.rel_grad_t.numpy()[g["rel_ids"].astype(np.int64)] = g["rel_rows"]
        return g["loss"]

    def zero_relation_grad(self):
        self.rel_grad_t.zero_()

    def relation_grad(self):
        return self.rel_grad_t

    def apply_relations(self):
        gr = self.rel_grad_t.numpy()
        ids = np.nonzero(np.any(gr != 0, axis=1))[0].astype(np.uint32)
        if len(ids):
            po.adagrad_apply(self.d, self.lr, self.eps, ids, gr[ids], self.rel_theta, self.rel_acc)

    def collective_stream(self):
        return contextlib.nullcontext()

    def after_handoff(self):
        pass
