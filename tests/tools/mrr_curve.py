#!/usr/bin/env python
"""Test- and train-edge MRR per epoch (unfiltered protocol, oracle evaluator) of GPU training on a
synthetic graph, for a list of learning rates: shows where the synthetic workloads' test MRR peaks and
that the later sag is over-fitting (train-edge MRR keeps rising). One JSON line per lr."""
import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)


def main():
    import torch

    import paper_2101_08358_b200 as eb
    from oracle import pyoracle as po
    ap = argparse.ArgumentParser()
    ap.add_argument("--V", type=int, default=420_000)
    ap.add_argument("--R", type=int, default=1)
    ap.add_argument("--E", type=int, default=6_000_000)
    ap.add_argument("--kind", default="dot")
    ap.add_argument("--dim", type=int, default=100)
    ap.add_argument("--b", type=int, default=50_000)
    ap.add_argument("--nt", type=int, default=100)
    ap.add_argument("--p", type=int, default=16)
    ap.add_argument("--epochs", type=int, default=5)
    ap.add_argument("--lrs", default="0.1,0.03,0.01")
    ap.add_argument("--test", type=int, default=20_000)
    a = ap.parse_args()
    edges, split = eb.generate_graph(a.V, a.R, a.E, seed=210108358, train_frac=0.9, valid_frac=0.05)
    train = edges[split == 0]
    test = edges[split == 2][:a.test]
    probe = train[np.random.default_rng(0).choice(len(train), a.test, replace=False)]
    bucketed, off = eb.bucket_edges(train, a.V, a.p)
    plan = eb.make_plan("elimination", a.p, a.p, 0)
    dev = torch.from_numpy(bucketed.view(np.int32)).cuda()
    for lr in [float(x) for x in a.lrs.split(",")]:
        h = eb.Hyper(kind=a.kind, dim=a.dim, lr=lr, batch_size=a.b, num_negatives=a.nt, alpha=0.5, neg_seed=1,
                     engine="tc")
        tr = eb.Trainer(h, a.V, a.R, a.p, device=0)
        tr.init_embeddings(11)
        rows = []
        for ep in range(a.epochs):
            loss = tr.train_epoch(dev, off, plan["seq"], ep)["loss"]
            th, _ = tr.node_table()
            rt = tr.relation_table()[0] if tr.rel_theta is not None else np.zeros((1, a.dim), np.float32)
            ev = lambda x: po.aggregate(po.eval_ranks(a.kind, a.dim, th, rt, a.V, x, train_edges=train,  # noqa: E731
                                                      n_eval_neg=1000, alpha_eval=0.5, block=1000, eval_seed=7))
            rows.append({"epoch": ep, "loss": round(loss, 4), "test_mrr": round(float(ev(test)["mrr"]), 5),
                         "train_mrr": round(float(ev(probe)["mrr"]), 5)})
        tr.close()
        print(json.dumps({"graph": {"V": a.V, "R": a.R, "E": a.E, "kind": a.kind, "dim": a.dim, "b": a.b,
                                    "nt": a.nt}, "lr": lr, "epochs": rows}), flush=True)


if __name__ == "__main__":
    main()
