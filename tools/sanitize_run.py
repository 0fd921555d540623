#!/usr/bin/env python
"""Small training workload for compute-sanitizer (memcheck / racecheck / synccheck / initcheck):
the tensor-core engine's kernels (TMA + mbarrier + tcgen05 pipelines, k_tc<ROWS/NEGS>, the fixup),
the cp.async-pipelined chain rule and segmented Adagrad, the gather/pack, sampling and key sort, eval,
the wide tensor-core path, the forced overflow repair, the multi-GPU relation path at world 1, plus
the partition buffer, at small sizes (several items per CTA through a capped grid)."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch

    import paper_2101_08358_b200 as eb
    V, R, p = 3000, 20, 2
    edges, split = eb.generate_graph(V, R, 12000, seed=5)
    bucketed, off = eb.bucket_edges(edges[split == 0], V, p)
    dev = torch.from_numpy(bucketed.view(np.int32)).cuda()
    plan = eb.make_plan("elimination", p, p, 0)
    for kind, dim, nt, b in (("complex", 100, 1000, 300), ("distmult", 32, 64, 256), ("dot", 128, 200, 200)):
        h = eb.Hyper(kind=kind, dim=dim, batch_size=b, num_negatives=nt, neg_seed=3, engine="tc")
        tr = eb.Trainer(h, V, R, p, device=0)
        tr.init_embeddings(11)
        tr.train_epoch(dev, off, plan["seq"], 0)
        bucket = dev[int(off[1]):int(off[2])]
        negs = tr.sample_negatives(bucket, 0, 1)
        tr.loss_and_grad(bucket[:b], negs, 0, 1)
        tr.eval_ranks(dev[:200], dev, n_eval=100, block=100)
        tr.synchronize()
        tr.close()
    # the wide tensor-core path (d > 128, chunked negatives), the overflow fixup forced on every row
    # (repaired inside the dN kernel), the multi-GPU relation path at world 1 (communication stream)
    for kind, dim, nt, b, chunks, env in (("complex", 160, 200, 256, 1, {}), ("distmult", 32, 64, 256, 2, {}),
                                          ("complex", 32, 64, 256, 1, {"EMBER_TC_ZMAX": "0"}),
                                          ("complex", 32, 64, 256, 1, {"EMBER_DENSE_RELATIONS": "1"})):
        os.environ.update(env)
        h = eb.Hyper(kind=kind, dim=dim, batch_size=b, num_negatives=nt, num_chunks=chunks, neg_seed=3, engine="tc")
        tr = eb.Trainer(h, V, R, p, device=0)
        tr.init_embeddings(11)
        tr.train_epoch(dev, off, plan["seq"], 0)
        tr.synchronize()
        tr.close()
        for k in env:
            del os.environ[k]
    # the (key, slot) sort on its own (bits 24 and 32)
    h = eb.Hyper(kind="complex", dim=16, batch_size=2000, num_negatives=100, neg_seed=3, engine="tc")
    tr = eb.Trainer(h, V, R, p, device=0)
    rng = np.random.default_rng(1)
    for bits in (24, 32):
        keys = rng.integers(0, 1 << 20, size=6000, dtype=np.int64).astype(np.uint32)
        tr.debug_sort_slots(torch.from_numpy(keys.view(np.int32)).cuda(), bits)
    tr.close()
    # the partition buffer (p=4, c=2)
    bucketed4, off4 = eb.bucket_edges(edges[split == 0], V, 4)
    dev4 = torch.from_numpy(bucketed4.view(np.int32)).cuda()
    plan4 = eb.make_plan("elimination", 4, 2, 0)
    h = eb.Hyper(kind="complex", dim=32, batch_size=256, num_negatives=64, neg_seed=3, engine="tc")
    tr = eb.Trainer(h, V, R, 4, device=0, allocate=False)
    buf = eb.PartitionBuffer(tr, 2, plan4["seq"])
    buf.init_backing(11)
    buf.train_epoch(dev4, off4, 0)
    buf.flush()
    buf.close()
    tr.close()
    print("sanitize workload done")


if __name__ == "__main__":
    main()
