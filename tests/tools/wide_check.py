#!/usr/bin/env python
"""Quick check of the d > 128 tensor-core path against the oracle (loss_and_grad at several shapes)."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


def main():
    import torch

    from gpu_helpers import host_tables, make_graph, make_trainer, oracle_model, rel_err, row_rel_err
    from oracle import pyoracle as po
    edges, off, _ = make_graph(V=3000, R=20, E=20000, p=2)
    bucket = edges[off[1]:off[2]]
    dev = lambda a: torch.from_numpy(np.ascontiguousarray(a).view(np.int32)).cuda()  # noqa: E731
    for kind, dim, nt, nb, ch in [("complex", 136, 100, 200, 1), ("distmult", 256, 300, 500, 1),
                                  ("complex", 800, 1000, 700, 1), ("dot", 144, 64, 129, 1), ("complex", 32, 64, 509, 4),
                                  ("distmult", 100, 200, 777, 3), ("complex", 800, 100, 300, 2), ("dot", 64, 40, 77, 2)]:
        tr = make_trainer(kind, dim=dim, b=max(nb, 16), nt=nt, p=2, chunks=ch, engine=os.environ.get("ENG", "tc"))
        th, _, rt, _ = host_tables(tr)
        negs = tr.sample_negatives(dev(bucket), 0, 1, 0, 0, 0)
        got = tr.loss_and_grad(dev(bucket[:nb]), negs, 0, 1)
        exp = po.loss_and_grad(oracle_model(tr), bucket[:nb], negs.cpu().numpy().view(np.uint32), th, rt)
        print(kind, dim, nt, nb, ch, "loss", got["loss"], exp["loss"], "lse", rel_err(got["lse"], exp["lse"]),
              "ids", bool((got["node_ids"] == exp["node_ids"]).all()),
              "rows", row_rel_err(got["node_rows"], exp["node_rows"]),
              "rel", row_rel_err(got["rel_rows"], exp["rel_rows"]) if kind != "dot" else 0.0, flush=True)
        tr.close()


if __name__ == "__main__":
    main()
