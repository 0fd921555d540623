#!/usr/bin/env python
"""End-to-end run at the Freebase86m shape on one B200: generate the graph, train whole epochs in
BETA order through the C-ABI (train_epoch_partitioned), and evaluate link prediction on the GPU
(unfiltered protocol: 1,000 sampled negatives per block of test edges, half degree-based,
PAPER.md:321). Prints one JSON line with the per-epoch loss, epoch time and MRR / Hits@k.

Usage: python tools/train_fb86m.py [--epochs 2] [--test 20000] [--config fb86m]
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch

    import bench
    import paper_2101_08358_b200 as eb

    ap = argparse.ArgumentParser()
    ap.add_argument("--epochs", type=int, default=2)
    ap.add_argument("--test", type=int, default=20000)
    ap.add_argument("--config", default="fb86m", choices=sorted(bench.CONFIGS))
    args = ap.parse_args()
    cfg = bench.CONFIGS[args.config]
    t0 = time.time()
    edges, split = eb.generate_graph(cfg["V"], cfg["R"], cfg["E"], bench.GRAPH_SEED, cfg["train"], cfg["valid"],
                                     device=0)
    test = edges[split == 2][: args.test].contiguous()
    train = edges[split == 0]
    del edges, split
    bucketed, offsets = eb.bucket_edges(train, cfg["V"], cfg["p"], device=0)
    del train
    torch.cuda.empty_cache()
    h = eb.Hyper(kind=cfg["kind"], dim=cfg["dim"], batch_size=cfg["b"], num_negatives=cfg["nt"], alpha=cfg["alpha"],
                 neg_seed=bench.NEG_SEED, engine="tc")
    tr = eb.Trainer(h, cfg["V"], cfg["R"], cfg["p"], device=0)
    tr.init_embeddings(bench.INIT_SEED)
    plan = eb.make_plan("elimination", cfg["p"], cfg["p"], bench.ORDER_SEED)
    setup_s = time.time() - t0

    # train edges ranked the same way: the test MRR's later sag with a rising train-edge MRR is
    # over-fitting of the synthetic graph (profiles/r02_mrr_curve_*.jsonl show the same on the CPU path)
    probe = bucketed[torch.randperm(bucketed.shape[0], device=bucketed.device)[: args.test]].contiguous()

    def evaluate(edges_eval=None):
        ranks = tr.eval_ranks(test if edges_eval is None else edges_eval, bucketed, n_eval=1000, alpha_eval=0.5,
                              block=1000, eval_seed=7)
        r = np.asarray(ranks, np.float64)  # MRR / Hits@k of the GPU ranks
        return {"mrr": float(np.mean(1.0 / r)), "hits@1": float(np.mean(r <= 1)), "hits@10": float(np.mean(r <= 10))}

    before = evaluate()
    epochs = []
    for ep in range(args.epochs):
        torch.cuda.synchronize()
        clocks = bench.ClockSampler(0)
        clocks.start()
        e0 = time.perf_counter()
        out = tr.train_epoch(bucketed, offsets, plan["seq"], ep)
        torch.cuda.synchronize()
        dt = time.perf_counter() - e0
        clk = clocks.stop()
        ovf = tr.overflow_rows()
        m = evaluate()
        mt = evaluate(probe)
        epochs.append({"epoch": ep, "loss": round(out["loss"], 4), "batches": int(out["batches"]),
                       "edges": int(out["edges"]), "seconds": round(dt, 3),
                       "edges_per_s": round(out["edges"] / dt, 1),
                       "mrr": round(float(m["mrr"]), 4), "hits@1": round(float(m["hits@1"]), 4),
                       "hits@10": round(float(m["hits@10"]), 4),
                       "train_edge_mrr": round(float(mt["mrr"]), 4),
                       "overflow_rows_total": int(ovf), "clocks": clk})
    print(json.dumps({"workload": cfg["desc"], "train_edges": int(offsets[-1]), "setup_s": round(setup_s, 1),
                      "eval": f"unfiltered, {args.test} test edges x 2 sides, 1000 sampled negatives per block of 1000",
                      "mrr_before": round(float(before["mrr"]), 4), "epochs": epochs}), flush=True)


if __name__ == "__main__":
    main()
