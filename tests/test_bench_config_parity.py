"""Parity at the benchmark's own configuration (BASELINE.json configs[2], bench.py's headline):
Freebase86m-shaped graph (86,054,151 nodes, 14,824 relations, 338.6 M edges, 16 partitions), ComplEx
d=100, b=5*10^4, n_t=10^3, the tensor-core engine, built exactly as bench.py builds it (bench.Workload)
and stepped through the batches bench.py times (from the middle of the epoch's BETA sequence).

For three consecutive steps, from the state the previous steps left:
  * negative ids bit-exact with the oracle's sampler;
  * loss_and_grad (C-ABI ember_loss_and_grad) against the CPU oracle on the compact parameter slice
    of the batch: loss, f_pos, lse, unique node/relation ids, gradient rows
    within 1e-4 relative (max-normalised and per row), and element-wise against a float64
    restatement (oracle/f64.py): every element within 1e-4 of its term magnitude M (the scale of any
    fp32 sum's rounding error) and within 1e-4 relative where the element is well conditioned;
  * the training step itself (C-ABI ember_train_batch, as bench.py calls it): the post-Adagrad
    theta/acc of every touched node row and relation row are BIT-IDENTICAL to the oracle's Adagrad
     applied to the pre-step rows with the step's gradient rows.
Statistics go to $EMBER_PARITY_OUT (JSON) when set (profiles/r02_parity_fb86m.json).
"""
import json
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import bench  # noqa: E402
import paper_2101_08358_b200 as eb  # noqa: E402
from oracle import f64  # noqa: E402
from oracle import pyoracle as po  # noqa: E402

from gpu_helpers import rel_err, row_rel_err  # noqa: E402

TOL = 1e-4  # north_star: per-step scores and gradients within 1e-4 relative


def _dev(a):
    return torch.from_numpy(np.ascontiguousarray(a, np.uint32).view(np.int32)).cuda()


@pytest.fixture(scope="module")
def workload():
    if torch.cuda.get_device_properties(0).total_memory < 120e9:
        pytest.skip("needs the full 68.8 GB FB86m-shaped tables in HBM")
    cfg = bench.CONFIGS["fb86m"]
    W = bench.Workload(cfg, 0, "tc")
    yield W
    W.tr.close()
    del W
    torch.cuda.empty_cache()


def test_fb86m_steps_match_oracle(workload):
    W = workload
    cfg, tr = W.cfg, W.tr
    V, p, d = cfg["V"], cfg["p"], cfg["dim"]
    m = po.model("complex", dim=d, lr=0.1, eps=1e-10, n_t=cfg["nt"], alpha=cfg["alpha"], chunks=1, seed=bench.NEG_SEED)
    first = len(W.batches) // 3 + 5  # bench.py's first timed batch (warm-up 5)
    report = {"config": cfg["desc"], "steps": []}
    for n in range(first, first + 3):
        lo, hi, begin, nb, i, j, step, k = W.batches[n]
        assert nb == cfg["b"]
        bucket_dev = W.edges[lo:hi]
        bucket = bucket_dev.cpu().numpy().view(np.uint32)
        oi, si, oj, sj = (eb.partition_offset(V, p, i), eb.partition_size(V, p, i), eb.partition_offset(V, p, j),
                          eb.partition_size(V, p, j))
        negs = tr.sample_negatives(bucket_dev, i, j, 0, step, k)
        negs_np = negs.cpu().numpy().view(np.uint32)
        assert (negs_np == po.sample_negatives(m, 0, step, k, bucket, oi, si, oj, sj)).all()
        batch = bucket[begin:begin + nb]
        ids = np.unique(np.concatenate([batch[:, 0], batch[:, 2], negs_np]))
        th_c, ac_c = (x.cpu().numpy() for x in tr.gather(_dev(ids), i, j))
        rt, ra = tr.relation_table()
        cb = np.stack([np.searchsorted(ids, batch[:, 0]), batch[:, 1], np.searchsorted(ids, batch[:, 2])], 1)
        cb = cb.astype(np.uint32)
        cn = np.searchsorted(ids, negs_np).astype(np.uint32)

        got = tr.loss_and_grad(_dev(batch), negs, i, j)
        exp = po.loss_and_grad(m, cb, cn, th_c, rt)
        x64 = f64.loss_and_grad("complex", cb, cn, th_c, rt)
        st = {"batch": n, "bucket": [i, j], "unique_node_rows": int(len(ids)),
              "unique_relations": int(len(exp["rel_ids"])), "loss_gpu": got["loss"], "loss_oracle": exp["loss"],
              "loss_f64": x64["loss"]}
        assert abs(got["loss"] - exp["loss"]) <= TOL * abs(exp["loss"])
        assert rel_err(got["fpos"], exp["fpos"]) <= TOL
        assert rel_err(got["lse"], exp["lse"]) <= TOL
        assert (got["node_ids"] == ids[exp["node_ids"]]).all()
        assert (got["rel_ids"] == exp["rel_ids"]).all()
        for name in ("node", "rel"):
            g, o, x, mag = got[f"{name}_rows"], exp[f"{name}_rows"], x64[f"{name}_rows"], x64[f"{name}_mag"]
            st[f"{name}_rows_rel_err_max_normalised"] = rel_err(g, o)
            st[f"{name}_rows_row_rel_err"] = row_rel_err(g, o)
            assert st[f"{name}_rows_rel_err_max_normalised"] <= TOL and st[f"{name}_rows_row_rel_err"] <= TOL
            eg, eo = f64.elementwise(g, x, mag), f64.elementwise(o, x, mag)
            st[f"{name}_rows_elementwise_gpu_vs_f64"] = eg
            st[f"{name}_rows_elementwise_oracle_vs_f64"] = eo
            assert eg["max_err_over_mag"] <= TOL, (name, eg)
            assert eg["max_rel_well_conditioned"] <= TOL, (name, eg)
        st["lse_max_abs_err_gpu_vs_f64"] = float(np.abs(got["lse"] - x64["lse"]).max())
        st["fpos_elementwise_gpu_vs_f64"] = f64.elementwise(got["fpos"], x64["fpos"], x64["fpos_mag"])
        st["fpos_elementwise_oracle_vs_f64"] = f64.elementwise(exp["fpos"], x64["fpos"], x64["fpos_mag"])
        assert st["fpos_elementwise_gpu_vs_f64"]["max_err_over_mag"] <= TOL

        # the training step through ember_train_batch: post-Adagrad rows bit-exact
        tr.train_batch(bucket_dev, begin, nb, i, j, 0, step, k)
        th_n, ac_n = (x.cpu().numpy() for x in tr.gather(_dev(ids), i, j))
        rt_n, ra_n = tr.relation_table()
        th_e, ac_e = th_c.copy(), ac_c.copy()
        po.adagrad_apply(d, 0.1, 1e-10, np.searchsorted(ids, got["node_ids"]).astype(np.uint32), got["node_rows"],
                         th_e, ac_e)
        po.adagrad_apply(d, 0.1, 1e-10, got["rel_ids"], got["rel_rows"], rt, ra)
        assert th_n.tobytes() == th_e.tobytes() and ac_n.tobytes() == ac_e.tobytes()
        assert rt_n.tobytes() == rt.tobytes() and ra_n.tobytes() == ra.tobytes()
        st["adagrad_bit_exact_rows"] = int(len(ids) + len(got["rel_ids"]))
        report["steps"].append(st)
    assert tr.overflow_rows() == 0
    out = os.environ.get("EMBER_PARITY_OUT")
    if out:
        json.dump(report, open(out, "w"), indent=1)
