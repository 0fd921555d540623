"""GPU parity through the C-ABI against the CPU oracle on identical seeded inputs.

Bars (BASELINE.json north_star): negative ids, init and bucket order bit-exact; per-step scores,
losses and gradients within 1e-4 relative (tolerance stated per assert); Adagrad bit-exact for
identical gradients.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2101_08358_b200 as eb  # noqa: E402
from oracle import pyoracle as po  # noqa: E402

from gpu_helpers import host_tables, make_graph, make_trainer, oracle_model, rel_err, row_rel_err  # noqa: E402

TOL = 1e-4  # per-step scores and gradients, relative (north_star)
ENGINES = ["simt", "tc"]


def _dev(a):
    return torch.from_numpy(np.ascontiguousarray(a).view(np.int32)).cuda()


@pytest.fixture(scope="module")
def graph():
    return make_graph(V=3000, R=20, E=20000, p=2)


def test_init_bit_exact_vs_oracle():
    tr = make_trainer("complex", dim=40, V=3000, p=2)
    th, ac, rt, _ = host_tables(tr)
    assert (ac == 0).all()
    ref = po.init_rows(11, 40, 0, 3000)
    assert th.tobytes() == ref.tobytes()
    assert rt.tobytes() == po.init_rows(11 ^ 0x52454C, 40, 0, 20).tobytes()


@pytest.mark.parametrize("chunks,alpha", [(1, 0.5), (3, 0.0), (2, 1.0)])
def test_negative_ids_bit_exact(graph, chunks, alpha):
    edges, off, _ = graph
    tr = make_trainer("distmult", nt=257, chunks=chunks, alpha=alpha, p=2)
    m = oracle_model(tr)
    for (i, j) in [(0, 0), (0, 1), (1, 0)]:
        b = i * 2 + j
        bucket = edges[off[b]:off[b + 1]]
        got = tr.sample_negatives(_dev(bucket), i, j, epoch=3, bucket_step=5, batch_in_bucket=7)
        exp = po.sample_negatives(m, 3, 5, 7, bucket, eb.partition_offset(3000, 2, i), eb.partition_size(3000, 2, i),
                                  eb.partition_offset(3000, 2, j), eb.partition_size(3000, 2, j))
        assert (got.cpu().numpy().view(np.uint32) == exp).all()


@pytest.mark.parametrize("engine", ENGINES)
@pytest.mark.parametrize("kind,chunks,nb", [("dot", 1, 512), ("distmult", 1, 512), ("complex", 1, 512),
                                            ("complex", 4, 509), ("distmult", 2, 77)])
def test_loss_and_grad_match_oracle(graph, engine, kind, chunks, nb):
    edges, off, _ = graph
    tr = make_trainer(kind, dim=32, nt=64, chunks=chunks, p=2, engine=engine)
    th, _, rt, _ = host_tables(tr)
    i, j = 0, 1
    bucket = edges[off[1]:off[2]]
    negs = tr.sample_negatives(_dev(bucket), i, j, 0, 0, 0)
    batch = bucket[:nb]
    got = tr.loss_and_grad(_dev(batch), negs, i, j)
    exp = po.loss_and_grad(oracle_model(tr), batch, negs.cpu().numpy().view(np.uint32), th, rt)
    assert abs(got["loss"] - exp["loss"]) <= TOL * abs(exp["loss"])
    assert rel_err(got["fpos"], exp["fpos"]) <= TOL
    assert rel_err(got["lse"], exp["lse"]) <= TOL
    assert (got["node_ids"] == exp["node_ids"]).all()
    assert row_rel_err(got["node_rows"], exp["node_rows"]) <= TOL
    assert rel_err(got["node_rows"], exp["node_rows"]) <= TOL
    assert (got["rel_ids"] == exp["rel_ids"]).all()
    if kind != "dot":
        assert row_rel_err(got["rel_rows"], exp["rel_rows"]) <= TOL


@pytest.mark.parametrize("engine", ["simt", "tc"])
@pytest.mark.parametrize("kind,dim,chunks,grid,zmax", [("complex", 800, 1, None, None), ("distmult", 256, 1, None, None),
                                                       ("dot", 132, 1, None, None), ("complex", 800, 3, "4", None),
                                                       ("complex", 160, 1, "3", "0"), ("distmult", 100, 2, None, None)])
def test_loss_and_grad_large_dim_and_chunks(graph, monkeypatch, engine, kind, dim, chunks, grid, zmax):
    """SURVEY config C5's d = 800 (and other d > 128) and chunked negative sets on the
    tensor-core engine's three-pass kernels (tc_wide.cu) and on the SIMT reference: scores, losses and
    gradients within 1e-4 of the oracle, including a capped grid (several items per CTA) and every row
    forced through the exact overflow recompute (EMBER_TC_ZMAX=0)."""
    if grid is not None:
        monkeypatch.setenv("EMBER_TC_MAXGRID", grid)
    if zmax is not None:
        monkeypatch.setenv("EMBER_TC_ZMAX", zmax)
    edges, off, _ = graph
    tr = make_trainer(kind, dim=dim, b=256, nt=100, chunks=chunks, p=2, engine=engine)
    th, _, rt, _ = host_tables(tr)
    bucket = edges[off[1]:off[2]]
    negs = tr.sample_negatives(_dev(bucket), 0, 1, 0, 0, 0)
    batch = bucket[:200]
    got = tr.loss_and_grad(_dev(batch), negs, 0, 1)
    exp = po.loss_and_grad(oracle_model(tr), batch, negs.cpu().numpy().view(np.uint32), th, rt)
    assert abs(got["loss"] - exp["loss"]) <= TOL * abs(exp["loss"])
    assert rel_err(got["lse"], exp["lse"]) <= TOL
    assert (got["node_ids"] == exp["node_ids"]).all()
    assert row_rel_err(got["node_rows"], exp["node_rows"]) <= TOL
    if kind != "dot":
        assert row_rel_err(got["rel_rows"], exp["rel_rows"]) <= TOL
    if zmax == "0" and engine == "tc":
        assert tr.overflow_rows() == 2 * 200  # every (row, side) took the exact path


def test_scores_match_oracle(graph):
    edges, off, _ = graph
    tr = make_trainer("complex", dim=32, nt=64, p=2)
    th, _, rt, _ = host_tables(tr)
    bucket = edges[off[1]:off[2]]
    negs = tr.sample_negatives(_dev(bucket), 0, 1)
    batch = bucket[:100]
    for side in (0, 1):
        got = tr.debug_scores(_dev(batch), negs, side=side, rows=50, i=0, j=1)
        nn = negs.cpu().numpy().view(np.uint32)[side * 64:(side + 1) * 64]
        exp = np.zeros((50, 64), np.float32)
        for r in range(50):
            s, rel, t = batch[r]
            for k in range(64):
                trip = (nn[k], rel, t) if side == 1 else (s, rel, nn[k])
                exp[r, k] = po.lib().orc_score(2, 32, th[trip[0]].copy(), rt[trip[1]].copy(), th[trip[2]].copy())
        assert rel_err(got, exp) <= TOL


def test_adagrad_bit_exact():
    tr = make_trainer("distmult", dim=32, p=1)
    th0, ac0, rt0, ra0 = host_tables(tr)
    rng = np.random.default_rng(0)
    ids = np.unique(rng.integers(0, 3000, 300)).astype(np.uint32)
    rows = rng.standard_normal((len(ids), 32)).astype(np.float32)
    tr.adagrad_apply(_dev(ids), torch.from_numpy(rows).cuda())
    tr.adagrad_apply(_dev(ids), torch.from_numpy(rows * 0.5).cuda())
    th, ac, _, _ = host_tables(tr)
    po.adagrad_apply(32, 0.1, 1e-10, ids, rows, th0, ac0)
    po.adagrad_apply(32, 0.1, 1e-10, ids, rows * 0.5, th0, ac0)
    assert th.tobytes() == th0.tobytes() and ac.tobytes() == ac0.tobytes()
    rid = np.array([0, 5, 19], np.uint32)
    rrows = rng.standard_normal((3, 32)).astype(np.float32)
    tr.adagrad_apply(_dev(rid), torch.from_numpy(rrows).cuda(), relations=True)
    po.adagrad_apply(32, 0.1, 1e-10, rid, rrows, rt0, ra0)
    _, _, rt, ra = host_tables(tr)
    assert rt.tobytes() == rt0.tobytes() and ra.tobytes() == ra0.tobytes()


def test_gather_parameter_slice():
    """ParameterSlice gather: one row per id, in id order, from partition i or j
    (or the relation table), bit-exact copies; an id outside both partitions is a ConfigError."""
    tr = make_trainer("complex", dim=40, V=3000, p=3)
    for k in range(3):  # non-zero acc rows
        lo, n = eb.partition_offset(3000, 3, k), eb.partition_size(3000, 3, k)
        ids_k = np.arange(lo, lo + n, 7, dtype=np.uint32)
        tr.adagrad_apply(_dev(ids_k), torch.ones((len(ids_k), 40), device="cuda"), k, k)
    with pytest.raises(eb.ConfigError):  # an id outside partitions i and j is rejected, not written
        tr.adagrad_apply(_dev(np.array([0], np.uint32)), torch.ones((1, 40), device="cuda"), 1, 2)
    th, ac, rt, ra = host_tables(tr)
    lo1, n1 = eb.partition_offset(3000, 3, 1), eb.partition_size(3000, 3, 1)
    lo2, n2 = eb.partition_offset(3000, 3, 2), eb.partition_size(3000, 3, 2)
    rng = np.random.default_rng(3)
    ids = np.concatenate([rng.integers(lo1, lo1 + n1, 200), rng.integers(lo2, lo2 + n2, 100), [lo1, lo2 + n2 - 1]])
    ids = ids.astype(np.uint32)
    gth, gac = tr.gather(_dev(ids), 1, 2)
    assert gth.cpu().numpy().tobytes() == th[ids].tobytes()
    assert gac.cpu().numpy().tobytes() == ac[ids].tobytes()
    gth, gac = tr.gather(_dev(ids[::-1].copy()), 2, 1, with_acc=False)
    assert gac is None and gth.cpu().numpy().tobytes() == th[ids[::-1]].tobytes()
    rid = np.array([19, 0, 7, 7], np.uint32)
    rth, rac = tr.gather(_dev(rid), relations=True)
    assert rth.cpu().numpy().tobytes() == rt[rid].tobytes() and rac.cpu().numpy().tobytes() == ra[rid].tobytes()
    with pytest.raises(eb.ConfigError):
        tr.gather(_dev(np.array([lo1, 0], np.uint32)), 1, 2)  # id 0 lives in partition 0
    with pytest.raises(eb.ConfigError):
        tr.gather(_dev(np.array([20], np.uint32)), relations=True)


@pytest.mark.parametrize("engine", ENGINES)
def test_non_finite_loss_is_an_error_naming_the_batch(graph, engine):
    """a non-finite score is an error carrying the batch id. The step records it on the
    device (no host sync in the step) and the next synchronising call returns status 2."""
    edges, off, _ = graph
    bucket = edges[off[1]:off[2]]
    tr = make_trainer("complex", dim=32, b=256, nt=64, p=2, engine=engine)
    tr.train_bucket(_dev(bucket), 0, 1, epoch=3, bucket_step=2)  # healthy: no error
    tr.synchronize()
    s = int(bucket[300, 0])  # source of an edge in batch 1 of the bucket (b = 256; batch 0 may draw it as a negative)
    tr.theta[0][s - eb.partition_offset(3000, 2, 0), 0] = float("nan")
    with pytest.raises(eb.EmberError, match=r"non-finite loss in batch \(epoch 4, bucket step 5, batch [01]\)"):
        tr.train_bucket(_dev(bucket), 0, 1, epoch=4, bucket_step=5)
    tr.synchronize()  # reported once


@pytest.mark.parametrize("engine,dim,chunks", [("simt", 32, 1), ("tc", 32, 1), ("tc", 160, 1), ("tc", 32, 2)])
def test_training_trajectory_matches_oracle(graph, engine, dim, chunks):
    """A few full steps (sample -> grads -> Adagrad) over two buckets; losses within 1e-4, tables
    close (Adagrad's first step is ~ -lr*sign(g), so elements whose gradient is at rounding level can
    legitimately flip: allow < 0.01% of elements)."""
    edges, off, _ = graph
    tr = make_trainer("complex", dim=dim, b=256, nt=64, chunks=chunks, p=2, engine=engine)
    th, ac, rt, ra = host_tables(tr)
    m = oracle_model(tr)
    V, p = 3000, 2
    for step, (i, j) in enumerate([(0, 1), (1, 1)]):
        b = i * p + j
        bucket = edges[off[b]:off[b + 1]]
        dbucket = _dev(bucket)
        loss_dev = torch.zeros(1, device="cuda")
        for k in range(2):
            tr.train_batch(dbucket, k * 256, 256, i, j, epoch=1, bucket_step=step, batch_in_bucket=k,
                           loss_out=loss_dev)
            tr.synchronize()  # the step runs on the context's own (non-blocking) stream
            l_gpu = float(loss_dev.item())
            l_cpu = po.train_batch(m, 1, step, k, bucket, k * 256, 256, eb.partition_offset(V, p, i),
                                   eb.partition_size(V, p, i), eb.partition_offset(V, p, j),
                                   eb.partition_size(V, p, j), th, ac, rt, ra)
            assert abs(l_gpu - l_cpu) <= TOL * abs(l_cpu), (step, k, l_gpu, l_cpu)
    gth, gac, grt, gra = host_tables(tr)
    for a, b_ in ((gth, th), (grt, rt)):
        bad = np.abs(a - b_) > 1e-3
        assert bad.sum() <= max(1, 1e-4 * bad.size), bad.sum()  # (the small relation table: one flip at most)
    assert rel_err(gac, ac) <= 1e-3 and rel_err(gra, ra) <= 1e-3


def test_eval_ranks_match_oracle(graph):
    edges, off, test = graph
    tr = make_trainer("distmult", dim=32, p=2)
    th, _, rt, _ = host_tables(tr)
    train = edges
    got = tr.eval_ranks(_dev(test), _dev(train), n_eval=200, alpha_eval=0.5, block=100, eval_seed=9)
    exp = po.eval_ranks("distmult", 32, th, rt, 3000, test, train_edges=train, n_eval_neg=200, alpha_eval=0.5,
                        block=100, eval_seed=9)
    assert (np.abs(got.astype(np.int64) - exp.astype(np.int64)) <= 1).mean() > 0.999
    a, b = po.aggregate(got), po.aggregate(exp)
    assert abs(a["mrr"] - b["mrr"]) < 1e-3


@pytest.mark.parametrize("kind,dim,nt,nb,zmax,grid", [("complex", 100, 1000, 3000, None, None),
                                                   ("complex", 100, 1000, 3000, None, "5"),
                                                   ("dot", 100, 1000, 1500, None, "2"),
                                                   ("distmult", 40, 100, 333, None, None),
                                                   ("complex", 64, 200, 700, "0", "3"),
                                                   ("distmult", 128, 300, 1000, None, "1"),
                                                   ("complex", 16, 17, 5, None, None)])
def test_tc_engine_headline_shapes(graph, monkeypatch, kind, dim, nt, nb, zmax, grid):
    """Tensor-core contraction at the headline d=100 / n_t=1000 shape (smaller b), ragged tiles
    (nb, n_t not multiples of the 128/64 tiles), d at the 128 limit, and zmax=0 (every row sent
    through the exact overflow fixup, k_tc_fixup), and capped grids (several items per CTA) — all within 1e-4 of the oracle."""
    if zmax is not None:
        monkeypatch.setenv("EMBER_TC_ZMAX", zmax)
    if grid is not None:  # few CTAs: every CTA walks several items (resident-operand hand-over)
        monkeypatch.setenv("EMBER_TC_MAXGRID", grid)
    edges, off, _ = graph
    tr = make_trainer(kind, dim=dim, b=max(nb, 16), nt=nt, p=2, engine="tc")
    th, _, rt, _ = host_tables(tr)
    bucket = edges[off[1]:off[2]]
    negs = tr.sample_negatives(_dev(bucket), 0, 1, 0, 0, 0)
    batch = bucket[:nb]
    got = tr.loss_and_grad(_dev(batch), negs, 0, 1)
    exp = po.loss_and_grad(oracle_model(tr), batch, negs.cpu().numpy().view(np.uint32), th, rt)
    assert abs(got["loss"] - exp["loss"]) <= TOL * abs(exp["loss"])
    assert rel_err(got["lse"], exp["lse"]) <= TOL
    assert (got["node_ids"] == exp["node_ids"]).all()
    assert row_rel_err(got["node_rows"], exp["node_rows"]) <= TOL
    if kind != "dot":
        assert row_rel_err(got["rel_rows"], exp["rel_rows"]) <= TOL


@pytest.mark.parametrize("kind,engine", [("complex", "tc"), ("distmult", "tc"), ("dot", "simt")])
def test_direct_unique_row_updates_bit_identical(graph, monkeypatch, kind, engine):
    """Node rows whose key occurs once in a batch are updated by their producer (chain rule / dN
    reduce) instead of the segmented reduction: parameters are bit-identical either way."""
    edges, off, _ = graph
    tabs = []
    for flag in ("0", "1"):
        monkeypatch.setenv("EMBER_NO_DIRECT", flag)
        tr = make_trainer(kind, dim=32, b=256, nt=64, p=2, engine=engine)
        for step, (i, j) in enumerate([(0, 1), (1, 1), (1, 0)]):
            b = i * 2 + j
            bucket = _dev(edges[off[b]:off[b + 1]])
            for k in range(3):
                tr.train_batch(bucket, k * 256, 256, i, j, epoch=0, bucket_step=step, batch_in_bucket=k)
        tabs.append(host_tables(tr))
        tr.close()
    for a, b_ in zip(tabs[0], tabs[1]):
        assert a.tobytes() == b_.tobytes()


@pytest.mark.parametrize("kind,b", [("complex", 256), ("distmult", 1500)])
def test_relation_first_reduction_bit_identical(graph, monkeypatch, kind, b):
    """The multi-GPU reduction order (relation keys reduced first into the dense buffer, their
    all-reduce + dense Adagrad on the communication stream while the node keys are reduced;
    EMBER_DENSE_RELATIONS=1 runs it at world 1) leaves every parameter bit-identical to the
    in-place single-launch reduction — hot relations and hub nodes (long segments) included."""
    edges, off, _ = graph
    tabs = []
    for flag in ("0", "1"):
        monkeypatch.setenv("EMBER_DENSE_RELATIONS", flag)
        tr = make_trainer(kind, dim=32, b=b, nt=64, p=2, engine="tc")
        for step, (i, j) in enumerate([(0, 1), (1, 1), (1, 0), (0, 0)]):
            bk = i * 2 + j
            bucket = _dev(edges[off[bk]:off[bk + 1]])
            n = (off[bk + 1] - off[bk]) // b
            for k in range(min(3, n)):
                tr.train_batch(bucket, k * b, b, i, j, epoch=0, bucket_step=step, batch_in_bucket=k)
        tr.synchronize()
        tabs.append(host_tables(tr))
        tr.close()
    for a, b_ in zip(tabs[0], tabs[1]):
        assert a.tobytes() == b_.tobytes()


@pytest.mark.parametrize("switch", ["EMBER_SAMPLE_ON_STEP", "EMBER_SEG_WALK", "EMBER_LONG_FINAL_LATE", "EMBER_DA_L2"])
def test_step_scheduling_switches_bit_identical(graph, monkeypatch, switch):
    """The step's scheduling choices leave every parameter bit-identical to their A/B alternative:
    negatives drawn by the packed gather while k_sample_keys runs on the helper stream (vs sampling
    on the step stream first), the segment kernel walking only the plan's runs with work (vs every
    run), k_long_final scheduled once the chunk partials exist (vs after the segment kernel), dA
    stored with an L2 evict_last policy (vs plain stores) — long segments included (b = 1500)."""
    edges, off, _ = graph
    tabs = []
    for on in (False, True):
        for sw in ("EMBER_SAMPLE_ON_STEP", "EMBER_SEG_WALK", "EMBER_LONG_FINAL_LATE", "EMBER_DA_L2"):
            monkeypatch.delenv(sw, raising=False)
        if on:
            monkeypatch.setenv(switch, "0" if switch == "EMBER_DA_L2" else "1")
        tr = make_trainer("distmult", dim=32, b=1500, nt=64, p=2, engine="tc")
        for step, (i, j) in enumerate([(0, 1), (1, 1), (1, 0), (0, 0)]):
            bk = i * 2 + j
            bucket = _dev(edges[off[bk]:off[bk + 1]])
            n = (off[bk + 1] - off[bk]) // 1500
            for k in range(min(3, n)):
                tr.train_batch(bucket, k * 1500, 1500, i, j, epoch=0, bucket_step=step, batch_in_bucket=k)
        tr.synchronize()
        tabs.append(host_tables(tr))
        tr.close()
    for a, b_ in zip(tabs[0], tabs[1]):
        assert a.tobytes() == b_.tobytes()


def test_host_batch_path_bit_identical(graph):
    """ember_train_batch_host (positives from pinned host memory, double-buffered asynchronous
    copies overlapping the previous step) trains exactly like ember_train_batch."""
    edges, off, _ = graph
    tabs = []
    keep = []  # pinned host batches must outlive their asynchronous copies
    for host in (False, True):
        tr = make_trainer("complex", dim=32, b=256, nt=64, p=2, engine="tc")
        for step, (i, j) in enumerate([(0, 1), (1, 1), (1, 0), (0, 0)]):
            b = i * 2 + j
            bucket_np = edges[off[b]:off[b + 1]]
            bucket = _dev(bucket_np)
            for k in range(3):
                if host:
                    hb = torch.from_numpy(np.ascontiguousarray(bucket_np[k * 256:(k + 1) * 256]).view(np.int32))
                    keep.append(hb.pin_memory())
                    loss = tr.train_batch_host(bucket, keep[-1], i, j, 0, step, k, want_loss=(k == 2))
                    if k == 2:
                        assert np.isfinite(loss)
                else:
                    tr.train_batch(bucket, k * 256, 256, i, j, 0, step, k)
        tabs.append(host_tables(tr))
        tr.close()
    for a, b_ in zip(tabs[0], tabs[1]):
        assert a.tobytes() == b_.tobytes()
