"""Pins the CPU oracle (oracle/ember_oracle.c) before anything is checked against it.

- RNG: bit-exact against the reference's own common.h (golden vectors produced by
  oracle/_ref, i.e. the unmodified reference sources compiled in place).
- model/eval ops: every SPEC worked example.
- gradients: central finite differences of an independent float64 numpy restatement
  of Eq. 2 (acceptance 7), >= 100 random d=8 cases, all kinds.
"""
import json
import math
import os

import numpy as np
import pytest

from oracle import pyoracle as po

GOLD = os.path.join(os.path.dirname(__file__), "golden")
REF = json.load(open(os.path.join(GOLD, "reference_rng_ordering.json")))
SPEC = json.load(open(os.path.join(GOLD, "spec_known_answers.json")))
L = po.lib()


# ------------------------------------------------------------------ RNG vs reference (common.h:51-117)

def test_splitmix_and_mix_seed_match_reference():
    for x, v in REF["splitmix64"].items():
        assert L.orc_splitmix64(int(x)) == v
    for k, v in REF["mix_seed"].items():
        a, b = map(int, k.split(","))
        assert L.orc_mix_seed(a, b) == v
    for k, v in REF["mix_seed3"].items():
        a, b, c = map(int, k.split(","))
        assert L.orc_mix_seed3(a, b, c) == v
    assert L.orc_mix_seed(0, 0x0E11) == 0x5531E629D8FBF9E6


@pytest.mark.parametrize("seed", list(REF["rng"].keys()))
def test_rng_streams_match_reference(seed):
    g = REF["rng"][seed]
    out = np.zeros(8, np.uint64)
    L.orc_rng_next(int(seed), 8, out)
    assert out.tolist() == g["next"]
    for n, exp in g["uniform_below"].items():
        L.orc_rng_uniform_below(int(seed), int(n), 8, out)
        assert out.tolist() == exp, n
    u = np.zeros(8, np.float32)
    L.orc_rng_uniform(int(seed), -0.1, 0.1, 8, u)
    assert u.view(np.uint32).tolist() == g["uniform_m0p1_0p1_bits"]


def test_rng_appendix_vectors():
    out = np.zeros(4, np.uint64)
    L.orc_rng_next(1, 4, out)
    assert [hex(x) for x in out.tolist()] == ["0x4bc8fde4f6ad0636", "0x8232dee91bc0acf3", "0xf02ded9ceb5676e0",
                                              "0x1c6b3433fd2f6929"]
    out = np.zeros(8, np.uint64)
    L.orc_rng_uniform_below(1, 1000, 8, out)
    assert out.tolist() == [296, 508, 938, 111, 148, 822, 111, 159]


# ------------------------------------------------------------------ partitions

def test_partition_geometry():
    assert [po.part_size(6, 2, k) for k in range(2)] == [3, 3]
    assert [po.part_size(7, 2, k) for k in range(2)] == [4, 3]
    assert po.part_offset(7, 2, 1) == 4
    V, p = 86_054_151, 16
    sizes = [po.part_size(V, p, k) for k in range(p)]
    assert sum(sizes) == V and max(sizes) - min(sizes) <= 1
    assert all(po.part_offset(V, p, k + 1) == po.part_offset(V, p, k) + sizes[k] for k in range(p - 1))


# ------------------------------------------------------------------ SPEC worked examples

def test_score_known_answers():
    s = np.array([1, 2], np.float32)
    d = np.array([3, 4], np.float32)
    one = np.ones(2, np.float32)
    assert L.orc_score(0, 2, s, one, d) == SPEC["score_dot_11"]["expect"]
    rng = np.random.default_rng(0)
    a, b = rng.standard_normal(8).astype(np.float32), rng.standard_normal(8).astype(np.float32)
    assert L.orc_score(1, 8, a, np.ones(8, np.float32), b) == pytest.approx(L.orc_score(0, 8, a, one[:1].repeat(8), b))
    # ComplEx with zero imaginary parts == DistMult on the real halves
    s4 = np.array([1.5, -2.0, 0, 0], np.float32)
    r4 = np.array([0.5, 3.0, 0, 0], np.float32)
    t4 = np.array([2.0, 1.0, 0, 0], np.float32)
    assert L.orc_score(2, 4, s4, r4, t4) == pytest.approx(L.orc_score(1, 2, s4[:2].copy(), r4[:2].copy(), t4[:2].copy()))


def test_adagrad_known_answers():
    th = np.zeros(1, np.float32)
    ac = np.zeros(1, np.float32)
    po.adagrad_apply(1, 0.1, 1e-10, [0], np.array([2.0], np.float32), th, ac)
    assert ac[0] == 4.0 and th[0] == pytest.approx(-0.1, abs=1e-7)
    th[:] = 0
    ac[:] = 0
    for _ in range(2):
        po.adagrad_apply(1, 0.1, 1e-10, [0], np.array([1.0], np.float32), th, ac)
    assert abs(th[0] - SPEC["adagrad_two"]["expect_theta"]) <= 1e-6
    th[:] = 0.3
    ac[:] = 0.7
    po.adagrad_apply(1, 0.1, 1e-10, [0], np.array([0.0], np.float32), th, ac)
    assert th[0] == np.float32(0.3) and ac[0] == np.float32(0.7)


def test_adagrad_disjoint_rows_commute_bitwise():
    rng = np.random.default_rng(3)
    th0 = rng.standard_normal((6, 4)).astype(np.float32)
    ac0 = np.abs(rng.standard_normal((6, 4))).astype(np.float32)
    g1 = rng.standard_normal((2, 4)).astype(np.float32)
    g2 = rng.standard_normal((2, 4)).astype(np.float32)
    a_th, a_ac, b_th, b_ac = th0.copy(), ac0.copy(), th0.copy(), ac0.copy()
    po.adagrad_apply(4, 0.1, 1e-10, [0, 3], g1, a_th, a_ac)
    po.adagrad_apply(4, 0.1, 1e-10, [1, 5], g2, a_th, a_ac)
    po.adagrad_apply(4, 0.1, 1e-10, [1, 5], g2, b_th, b_ac)
    po.adagrad_apply(4, 0.1, 1e-10, [0, 3], g1, b_th, b_ac)
    assert a_th.tobytes() == b_th.tobytes() and a_ac.tobytes() == b_ac.tobytes()


def _tiny_graph(kind, d, nb=5, V=12, R=3, nt=4, seed=0):
    rng = np.random.default_rng(seed)
    edges = np.stack([rng.integers(0, V, nb), rng.integers(0, R, nb), rng.integers(0, V, nb)], 1).astype(np.uint32)
    theta = (rng.standard_normal((V, d)) * 0.5).astype(np.float32)
    rel = (rng.standard_normal((R, d)) * 0.5).astype(np.float32)
    negs = rng.integers(0, V, 2 * nt).astype(np.uint32)
    return edges, theta, rel, negs


def test_loss_known_answers():
    # one positive, zero negatives -> loss exactly 0
    edges, theta, rel, _ = _tiny_graph("distmult", 4, nb=1, nt=0)
    m = po.model("distmult", dim=4, n_t=0)
    out = po.loss_and_grad(m, edges, np.zeros(0, np.uint32), theta, rel)
    assert out["loss"] == 0.0
    # all scores zero, n negatives -> log(1+n) per side
    for n in (1, 5, 1000):
        m = po.model("dot", dim=4, n_t=n)
        th = np.zeros((10, 4), np.float32)
        e = np.array([[1, 0, 2], [3, 0, 4]], np.uint32)
        out = po.loss_and_grad(m, e, np.zeros(2 * n, np.uint32) + 5, th, np.zeros((1, 4), np.float32))
        assert out["loss"] == pytest.approx(2 * math.log(1 + n), rel=1e-6)


def test_loss_invariant_to_negative_order():
    edges, theta, rel, negs = _tiny_graph("complex", 8, nt=6)
    m = po.model("complex", dim=8, n_t=6)
    a = po.loss_and_grad(m, edges, negs, theta, rel)
    perm = np.concatenate([np.random.default_rng(1).permutation(6), 6 + np.random.default_rng(2).permutation(6)])
    b = po.loss_and_grad(m, edges, negs[perm], theta, rel)
    assert a["loss"] == pytest.approx(b["loss"], rel=1e-6)


# ------------------------------------------------------------------ finite differences

def np_loss64(kind, edges, negs, theta, rel, chunks=1):
    """Independent float64 restatement of Eq. 2 (sign per SPEC.md:192)."""
    theta = theta.astype(np.float64)
    rel = rel.astype(np.float64)
    nb = len(edges)
    d = theta.shape[1]
    h = d // 2
    nt = len(negs) // (2 * chunks)
    rows = -(-nb // chunks)

    def f(s, r, t):
        if kind == "dot":
            return s @ t
        if kind == "distmult":
            return np.sum(s * r * t, -1)
        sc = s[..., :h] + 1j * s[..., h:]
        rc = r[..., :h] + 1j * r[..., h:]
        tc = t[..., :h] + 1j * t[..., h:]
        return np.real(np.sum(sc * rc * np.conj(tc), -1))

    total = 0.0
    for e, (s, r, t) in enumerate(edges):
        q = e // rows
        pos = f(theta[s], rel[r], theta[t])
        for side in (0, 1):
            ng = negs[(q * 2 + side) * nt:(q * 2 + side + 1) * nt]
            if side == 0:
                sc = np.array([f(theta[s], rel[r], theta[x]) for x in ng])
            else:
                sc = np.array([f(theta[x], rel[r], theta[t]) for x in ng])
            allv = np.concatenate([[pos], sc])
            mx = allv.max()
            total += -pos + mx + math.log(np.exp(allv - mx).sum())
    return total / nb


@pytest.mark.parametrize("kind", ["dot", "distmult", "complex"])
def test_gradients_match_finite_differences(kind):
    d, hstep = 8, 1e-4
    worst = 0.0
    for trial in range(34):  # 3 kinds x 34 = 102 random d=8 cases
        chunks = 1 + (trial % 2)
        edges, theta, rel, _ = _tiny_graph(kind, d, nb=4, V=9, R=2, nt=3, seed=100 + trial)
        negs = np.random.default_rng(trial).integers(0, 9, 2 * 3 * chunks).astype(np.uint32)
        m = po.model(kind, dim=d, n_t=3, chunks=chunks)
        out = po.loss_and_grad(m, edges, negs, theta, rel)
        assert out["loss"] == pytest.approx(np_loss64(kind, edges, negs, theta, rel, chunks), rel=1e-5)
        # node gradients
        for i, nid in enumerate(out["node_ids"]):
            fd = np.zeros(d)
            for k in range(d):
                tp, tm = theta.astype(np.float64), theta.astype(np.float64)
                tp = tp.copy(); tm = tm.copy()
                tp[nid, k] += hstep
                tm[nid, k] -= hstep
                fd[k] = (np_loss64(kind, edges, negs, tp, rel, chunks) - np_loss64(kind, edges, negs, tm, rel, chunks)) / (2 * hstep)
            err = np.abs(out["node_rows"][i] - fd).max() / max(np.abs(fd).max(), 1e-3)
            worst = max(worst, err)
            assert err <= 1e-4, (kind, trial, nid, out["node_rows"][i], fd)
        for i, rid in enumerate(out["rel_ids"]):
            fd = np.zeros(d)
            for k in range(d):
                rp = rel.astype(np.float64).copy(); rm = rp.copy()
                rp[rid, k] += hstep
                rm[rid, k] -= hstep
                fd[k] = (np_loss64(kind, edges, negs, theta, rp, chunks) - np_loss64(kind, edges, negs, theta, rm, chunks)) / (2 * hstep)
            err = np.abs(out["rel_rows"][i] - fd).max() / max(np.abs(fd).max(), 1e-3)
            assert err <= 1e-4, (kind, trial, rid)
        # touched rows are exactly the batch rows
        touched = set(edges[:, 0]) | set(edges[:, 2]) | set(negs.tolist())
        assert set(out["node_ids"].tolist()) == touched
    assert worst <= 1e-4


# ------------------------------------------------------------------ sampling

def _bucket(n=2000, V=100, seed=0):
    rng = np.random.default_rng(seed)
    return np.stack([rng.integers(0, V, n), np.zeros(n, int), rng.integers(0, V, n)], 1).astype(np.uint32)


def test_sampler_alpha0_uniform_over_partition():
    m = po.model("dot", n_t=1000, alpha=0.0, seed=5)
    out = po.sample_negatives(m, 0, 0, 0, _bucket(), 10, 20, 40, 30)
    dst, src = out[:1000], out[1000:]
    assert dst.min() >= 40 and dst.max() < 70 and src.min() >= 10 and src.max() < 30
    # chi-square uniformity over the 30-row dst pool
    cnt = np.bincount(dst - 40, minlength=30)
    chi2 = ((cnt - 1000 / 30) ** 2 / (1000 / 30)).sum()
    assert chi2 < 70  # df=29, p~1e-4


def test_sampler_degree_ratio_9_to_1():
    # alpha=1, degrees (9,1) over 2 nodes -> 9:1 within 3 sigma over 1e5 draws
    edges = np.array([[0, 0, 0]] * 9 + [[1, 0, 1]], np.uint32)
    tot = np.zeros(2)
    m = po.model("dot", n_t=1000, alpha=1.0, seed=11)
    for b in range(100):
        out = po.sample_negatives(m, 0, 0, b, edges, 0, 2, 0, 2)[:1000]
        tot += np.bincount(out, minlength=2)
    n = tot.sum()
    p = tot[0] / n
    assert n == 100_000 and abs(p - 0.9) <= 3 * math.sqrt(0.9 * 0.1 / n)


def test_sampler_deterministic_and_counter_based():
    m = po.model("dot", n_t=50, alpha=0.5, chunks=3, seed=9)
    b = _bucket()
    a1 = po.sample_negatives(m, 2, 7, 3, b, 0, 100, 0, 100)
    a2 = po.sample_negatives(m, 2, 7, 3, b, 0, 100, 0, 100)
    a3 = po.sample_negatives(m, 2, 7, 4, b, 0, 100, 0, 100)
    assert (a1 == a2).all() and not (a1 == a3).all()
    assert a1.size == 3 * 2 * 50
    # slot 0 of (chunk 0, side 0) is exactly Rng(mix_seed(mix_seed(mix_seed(seed,epoch,step),batch), 0)).uniform_below(n_bucket) -> dst
    base = L.orc_mix_seed(L.orc_mix_seed3(9, 2, 7), 3)
    draw = np.zeros(1, np.uint64)
    L.orc_rng_uniform_below(L.orc_mix_seed(base, 0), len(b), 1, draw)
    assert a1[0] == b[int(draw[0]), 2]


# ------------------------------------------------------------------ init

def test_init_range_determinism_and_mean():
    t1 = po.init_rows(3, 100, 0, 10_000)
    t2 = po.init_rows(3, 100, 0, 10_000)
    assert t1.tobytes() == t2.tobytes()
    assert np.abs(t1).max() <= np.float32(0.1)
    sigma = 0.1 / math.sqrt(3) / math.sqrt(t1.size)
    assert abs(t1.mean()) <= 3 * sigma
    # rows are independent streams: a slice equals the same rows generated standalone
    assert po.init_rows(3, 100, 500, 10).tobytes() == t1[500:510].tobytes()


# ------------------------------------------------------------------ eval

def test_eval_aggregate_and_ties():
    agg = po.aggregate(np.array([1, 2, 4], np.uint32), ks=(1, 10))
    assert agg["mrr"] == pytest.approx(SPEC["eval_mrr"]["mrr"]) and agg["hits@1"] == pytest.approx(1 / 3)
    assert agg["hits@10"] == 1.0
    # pessimistic tie: positive tied with 2 negatives, above the rest -> rank 3
    # DistMult d=2 with r=[1,-1], s=[1,1] so the source itself scores 0 as a candidate.
    theta = np.array([[1, 1], [0.5, 0], [0.5, 0], [0.5, 0], [0.1, 0], [-1, 0]], np.float32)
    rel = np.array([[1, -1]], np.float32)
    test = np.array([[0, 0, 1]], np.uint32)
    ranks = po.eval_ranks("distmult", 2, theta, rel, 6, test, filtered=True, filter_keys=po.pack_keys(test))
    assert ranks[0] == 3
    # filtered: a true triple among candidates is dropped
    keys = po.pack_keys(np.array([[0, 0, 1], [0, 0, 2]], np.uint32))
    ranks = po.eval_ranks("distmult", 2, theta, rel, 6, test, filtered=True, filter_keys=keys)
    assert ranks[0] == 2


def test_eval_monotone_in_negatives():
    rng = np.random.default_rng(0)
    theta = rng.standard_normal((50, 4)).astype(np.float32)
    test = np.stack([rng.integers(0, 50, 20), np.zeros(20, int), rng.integers(0, 50, 20)], 1).astype(np.uint32)
    r1 = po.eval_ranks("dot", 4, theta, np.zeros((1, 4), np.float32), 50, test, train_edges=test, n_eval_neg=10,
                       alpha_eval=0.0, block=20)
    r2 = po.eval_ranks("dot", 4, theta, np.zeros((1, 4), np.float32), 50, test, train_edges=test, n_eval_neg=40,
                       alpha_eval=0.0, block=20)
    assert (r2 >= 1).all() and r2.mean() >= r1.mean()


def test_graph_generator_restatement_matches_product_generator():
    """bench.py's CPU arm builds its graph with the oracle's restatement of the benchmark generator
    (orc_graph_generate / orc_graph_bucket); it must give the product generator's graph exactly."""
    import paper_2101_08358_b200 as eb
    V, R = 86_054_151, 14_824
    e1, s1 = po.graph_generate(V, R, 300_000, 210108358, 0.9, 0.05, first=12_345)
    e2, s2 = eb.generate_graph(V, R, 312_345, 210108358, 0.9, 0.05)
    assert np.array_equal(e1, e2[12_345:]) and np.array_equal(s1, s2[12_345:])
    b1, o1 = po.graph_bucket(V, 16, e1, s1, 0)
    b2, o2 = eb.bucket_edges(e2[12_345:][s2[12_345:] == 0], V, 16)
    assert np.array_equal(b1, b2) and np.array_equal(o1, o2)
    e3, _ = po.graph_generate(4_847_571, 1, 50_000, 7)
    e4, _ = eb.generate_graph(4_847_571, 1, 50_000, 7)
    assert np.array_equal(e3, e4)


@pytest.mark.parametrize("kind,chunks", [("dot", 1), ("distmult", 2), ("complex", 1), ("complex", 3)])
def test_float64_yardstick_matches_oracle(kind, chunks):
    """oracle/f64.py (the float64 restatement the full-size GPU parity test measures element-wise
    errors against) agrees with the C oracle on the same inputs."""
    from oracle import f64
    rng = np.random.default_rng(1)
    V, R, d, nb, nt = 400, 7, 24, 90, 16
    th = (rng.standard_normal((V, d)) * 0.4).astype(np.float32)
    rt = (rng.standard_normal((R, d)) * 0.4).astype(np.float32)
    e = np.stack([rng.integers(0, V, nb), rng.integers(0, R, nb), rng.integers(0, V, nb)], 1).astype(np.uint32)
    negs = rng.integers(0, V, chunks * 2 * nt).astype(np.uint32)
    a = po.loss_and_grad(po.model(kind, dim=d, n_t=nt, chunks=chunks), e, negs, th, rt)
    b = f64.loss_and_grad(kind, e, negs, th, rt, chunks=chunks)
    assert abs(a["loss"] - b["loss"]) <= 1e-6 * abs(b["loss"])
    assert np.abs(a["lse"].reshape(2, -1) - b["lse"]).max() <= 1e-5
    assert (a["node_ids"] == b["node_ids"]).all() and (a["rel_ids"] == b["rel_ids"]).all()
    st = f64.elementwise(a["node_rows"], b["node_rows"], b["node_mag"])
    assert st["max_err_over_mag"] <= 1e-6, st
    if kind != "dot":
        assert f64.elementwise(a["rel_rows"], b["rel_rows"], b["rel_mag"])["max_err_over_mag"] <= 1e-6
