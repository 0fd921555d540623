"""The reference-shaped C++ surface (include/ember/model.h, config.h, pipeline.h — ModelKind,
NegativeSampleSpec, ParameterSlice, GradientDelta, RunConfig, score, sample_negatives, loss_and_grad,
adagrad_step, init_embeddings, train_epoch_sync, train_epoch_partitioned; SPEC.md:116-206, 359-435,
504-507) compiled with g++ as a C++ consumer would, linked against libember_b200.so, and checked:
  * CPU: RunConfig validation raises ConfigError for every SPEC invariant violation; score() known
    answers;
  * GPU: one batch through sample_negatives -> loss_and_grad -> adagrad_step against the CPU oracle
    (negative ids bit-exact, loss/gradients within 1e-4, Adagrad bit-exact), a train_epoch_sync epoch
    with its loss against the oracle's sync trainer and its tables bit-identical to the Python host
    mirror's epoch, and train_epoch_partitioned through the partition buffer (p=4, c=2) bit-identical
    to the all-resident run (c=4) with misses = plan swap_count.
"""
import os
import subprocess

import numpy as np
import pytest

import paper_2101_08358_b200 as eb
from oracle import pyoracle as po
from paper_2101_08358_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
TOL = 1e-4


def _build(tmp_path):
    exe = tmp_path / "train_cpp"
    libdir = os.path.dirname(_lib.LIB_PATH)
    cc = "/usr/bin/g++" if os.path.exists("/usr/bin/g++") else "g++"
    subprocess.run([cc, "-std=c++17", "-O1", "-Wall", "-Werror", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "cpp", "train_cpp.cpp"), "-o", str(exe), f"-L{libdir}",
                    "-l:libember_b200.so", f"-Wl,-rpath,{libdir}"], check=True)
    return exe


def test_cpp_api_compiles_and_validates(tmp_path):
    exe = _build(tmp_path)
    r = subprocess.run([str(exe), "cpu"], capture_output=True, text=True, timeout=60)
    assert r.returncode == 0 and "cpu ok (0 failures)" in r.stdout, r.stdout + r.stderr


@pytest.mark.gpu
def test_cpp_api_trains_like_the_oracle(tmp_path):
    torch = pytest.importorskip("torch")
    exe = _build(tmp_path)
    out = tmp_path / "out"
    out.mkdir()
    r = subprocess.run([str(exe), "gpu", str(out)], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0 and "gpu ok (0 failures)" in r.stdout, r.stdout + r.stderr

    def ld(name, dt=np.float32):
        return np.fromfile(out / f"{name}.bin", dtype=dt)

    V, R, d, nt, b = 3000, 20, 32, 64, 256
    m = po.model("complex", dim=d, lr=0.1, eps=1e-10, n_t=nt, alpha=0.5, chunks=1, seed=3)
    edges = ld("edges_p2", np.uint32).reshape(-1, 3)
    off = ld("offsets_p2", np.uint64)
    th0 = np.concatenate([ld("theta0_p0"), ld("theta0_p1")]).reshape(V, d)
    rt0 = ld("rel0").reshape(R, d)
    assert th0.tobytes() == po.init_rows(11, d, 0, V).tobytes()  # init_embeddings bit-exact
    bucket = edges[off[1]:off[2]]
    negs = ld("negs", np.uint32)
    assert (negs == po.sample_negatives(m, 0, 0, 0, bucket, 0, 1500, 1500, 1500)).all()
    exp = po.loss_and_grad(m, bucket[:b], negs, th0, rt0)
    loss = float(ld("loss", np.float64)[0])
    assert abs(loss - exp["loss"]) <= TOL * abs(exp["loss"])
    ids, rows = ld("node_ids", np.uint32), ld("node_rows").reshape(-1, d)
    assert (ids == exp["node_ids"]).all()
    assert np.abs(rows - exp["node_rows"]).max() <= TOL * np.abs(exp["node_rows"]).max()
    rids, rrows = ld("rel_ids", np.uint32), ld("rel_rows").reshape(-1, d)
    assert (rids == exp["rel_ids"]).all()
    assert np.abs(rrows - exp["rel_rows"]).max() <= TOL * np.abs(exp["rel_rows"]).max()
    # adagrad_step applied the library's own GradientDelta: bit-exact vs the oracle's Adagrad
    th_e, ac_e, rt_e, ra_e = th0.copy(), np.zeros_like(th0), rt0.copy(), np.zeros_like(rt0)
    po.adagrad_apply(d, 0.1, 1e-10, ids, rows, th_e, ac_e)
    po.adagrad_apply(d, 0.1, 1e-10, rids, rrows, rt_e, ra_e)
    assert np.concatenate([ld("theta1_p0"), ld("theta1_p1")]).tobytes() == th_e.tobytes()
    assert np.concatenate([ld("acc1_p0"), ld("acc1_p1")]).tobytes() == ac_e.tobytes()
    assert ld("rel1").tobytes() == rt_e.tobytes()

    # train_epoch_sync: the same epoch through the Python host mirror is bit-identical; the loss matches
    # the oracle's sync trainer on the same batches
    h = eb.Hyper(kind="complex", dim=d, batch_size=b, num_negatives=nt, alpha=0.5, neg_seed=3, engine="tc")
    tr = eb.Trainer(h, V, R, 2, device=0)
    tr.init_embeddings(11)
    ids_d = torch.from_numpy(ids.view(np.int32)).cuda()
    tr.adagrad_apply(ids_d, torch.from_numpy(rows).cuda(), 0, 1)
    tr.adagrad_apply(torch.from_numpy(rids.view(np.int32)).cuda(), torch.from_numpy(rrows).cuda(), relations=True)
    plan = eb.make_plan("elimination", 2, 2, 0)
    py = tr.train_epoch(torch.from_numpy(edges.view(np.int32)).cuda(), off, plan["seq"], 0)
    th_py, _ = tr.node_table()
    assert np.concatenate([ld("theta2_p0"), ld("theta2_p1")]).tobytes() == th_py.tobytes()
    assert ld("rel2").tobytes() == tr.relation_table()[0].tobytes()
    assert float(ld("epoch_loss_p2", np.float64)[0]) == pytest.approx(py["loss"], rel=1e-12)
    tr.close()
    ls = []
    for step, (i, j) in enumerate(plan["seq"]):
        i, j = int(i), int(j)
        lo, hi = int(off[i * 2 + j]), int(off[i * 2 + j + 1])
        for k, b0 in enumerate(range(0, hi - lo, b)):
            ls.append(po.train_batch(m, 0, step, k, edges[lo:hi], b0, min(b, hi - lo - b0),
                                     eb.partition_offset(V, 2, i), eb.partition_size(V, 2, i),
                                     eb.partition_offset(V, 2, j), eb.partition_size(V, 2, j), th_e, ac_e, rt_e,
                                     ra_e))
    assert float(ld("epoch_loss_p2", np.float64)[0]) == pytest.approx(float(np.mean(ls)), rel=1e-3)

    # train_epoch_partitioned through the buffer (c=2 of p=4) == all partitions resident (c=4)
    assert ld("theta_p4_c2").tobytes() == ld("theta_p4_c4").tobytes()
    assert ld("rel_p4_c2").tobytes() == ld("rel_p4_c4").tobytes()
    assert (ld("loss_p4_c2", np.float64) == ld("loss_p4_c4", np.float64)).all()
    ref_plan = po.ref_plan(0, 4, 2, 0)  # the reference's own make_plan
    assert (ld("plan_p4c2", np.uint32).reshape(-1, 2) == ref_plan["seq"]).all()
