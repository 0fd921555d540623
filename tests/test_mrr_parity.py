"""End-to-end parity (BASELINE.json north_star): final MRR and Hits@10 of a model trained on the
GPU match the CPU reference path (the oracle, oracle/ember_oracle.c) within 0.005 absolute.

Both trainers consume the same bucket sequence (BETA plan), the same seeded negatives
(bit-exact sampler) and the same initial parameters (bit-exact init); per-step arithmetic
agrees to ~1e-5 relative (bf16x3 tensor cores vs fp32), so the trajectories stay close and the
ranking metrics agree. Both parameter sets are ranked by the same evaluator (the oracle's
filtered protocol: every node is a candidate, known true edges are filtered,
pessimistic ties), so the comparison isolates training.

Cases: a small DistMult graph, a 2-partition ComplEx graph, the FB15k-237-shaped config C1
at full shape (14,541 nodes, 237 relations, d=100, b=10^4, n_t=10^3), and a d=160
ComplEx graph (d > 128: the tensor-core engine's three-pass kernels, tc_wide.cu).
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2101_08358_b200 as eb  # noqa: E402
from oracle import pyoracle as po  # noqa: E402

TOL_MRR = 0.005  # north_star: MRR and Hits@10 within 0.005 absolute

CASES = {
    "small-distmult": dict(kind="distmult", V=3000, R=30, E=60000, d=32, p=1, b=1000, nt=100, epochs=6, n_test=2000,
                           seed=21),
    "complex-p2": dict(kind="complex", V=4000, R=20, E=80000, d=48, p=2, b=1500, nt=200, epochs=5, n_test=2000,
                       seed=22),
    "fb15k237-shape": dict(kind="distmult", V=14541, R=237, E=340144, d=100, p=1, b=10000, nt=1000, epochs=3,
                           n_test=5000, seed=210108358),
    # d > 128: the tensor-core engine's three-pass kernels (tc_wide.cu)
    "complex-p2-d160": dict(kind="complex", V=4000, R=20, E=80000, d=160, p=2, b=1500, nt=200, epochs=3,
                            n_test=2000, seed=23),
}


@pytest.mark.parametrize("case", list(CASES))
def test_trained_mrr_matches_cpu_reference(case):
    c = CASES[case]
    V, R, d, p, B = c["V"], c["R"], c["d"], c["p"], c["b"]
    edges, split = eb.generate_graph(V, R, c["E"], seed=c["seed"], train_frac=0.8, valid_frac=0.1)
    train = edges[split == 0]
    test = edges[split == 2][: c["n_test"]]
    bucketed, off = eb.bucket_edges(train, V, p)
    plan = eb.make_plan("elimination", p, p, 0)

    # GPU (the product path, tensor-core engine)
    h = eb.Hyper(kind=c["kind"], dim=d, batch_size=B, num_negatives=c["nt"], alpha=0.5, neg_seed=1,
                 engine=c.get("engine", "tc"))
    tr = eb.Trainer(h, V, R, p, device=0)
    tr.init_embeddings(11)
    dev = torch.from_numpy(bucketed.view(np.int32)).cuda()
    g_loss = [tr.train_epoch(dev, off, plan["seq"], ep)["loss"] for ep in range(c["epochs"])]
    g_th, _ = tr.node_table()
    g_rt = tr.relation_table()[0] if tr.rel_theta is not None else np.zeros((1, d), np.float32)

    # CPU reference path (oracle), same batches in the same order
    m = po.model(c["kind"], dim=d, lr=0.1, eps=1e-10, n_t=c["nt"], alpha=0.5, chunks=1, seed=1)
    th = po.init_rows(11, d, 0, V)
    ac = np.zeros_like(th)
    rt = po.init_rows(11 ^ 0x52454C, d, 0, R)
    ra = np.zeros_like(rt)
    c_loss = []
    for ep in range(c["epochs"]):
        ls = []
        for step, (i, j) in enumerate(plan["seq"]):
            i, j = int(i), int(j)
            lo, hi = int(off[i * p + j]), int(off[i * p + j + 1])
            bucket = bucketed[lo:hi]
            for k, b0 in enumerate(range(0, hi - lo, B)):
                ls.append(po.train_batch(m, ep, step, k, bucket, b0, min(B, hi - lo - b0),
                                         eb.partition_offset(V, p, i), eb.partition_size(V, p, i),
                                         eb.partition_offset(V, p, j), eb.partition_size(V, p, j), th, ac, rt, ra))
        c_loss.append(float(np.mean(ls)))
    assert np.allclose(g_loss, c_loss, rtol=1e-4), (g_loss, c_loss)

    keys = po.pack_keys(edges)
    gm = po.aggregate(po.eval_ranks(c["kind"], d, g_th, g_rt, V, test, filtered=True, filter_keys=keys))
    cm = po.aggregate(po.eval_ranks(c["kind"], d, th, rt, V, test, filtered=True, filter_keys=keys))
    assert cm["mrr"] > 20.0 / V, "the planted structure must be learnt (MRR far above random)"
    assert abs(gm["mrr"] - cm["mrr"]) <= TOL_MRR, (gm, cm)
    assert abs(gm["hits@10"] - cm["hits@10"]) <= TOL_MRR, (gm, cm)

    # the GPU evaluator on the GPU-trained tables agrees with the CPU evaluator (filtered protocol)
    fk = torch.from_numpy(keys.view(np.int64)).cuda()
    got = tr.eval_ranks_filtered(torch.from_numpy(np.ascontiguousarray(test).view(np.int32)).cuda(), fk)
    exp = po.eval_ranks(c["kind"], d, g_th, g_rt, V, test, filtered=True, filter_keys=keys)
    a, b = po.aggregate(got), po.aggregate(exp)
    assert abs(a["mrr"] - b["mrr"]) <= 1e-3 and abs(a["hits@10"] - b["hits@10"]) <= 1e-3, (a, b)
    tr.close()
