"""Multi-GPU path on CPU: the conflict-free round schedule (C-ABI, host code) and the
DistributedTrainer orchestration (lockstep relation all-reduce, P2P partition handoff) with gloo,
world_size 2, over the CPU oracle backend (tests/dist_oracle_backend.py).

Bars: the schedule covers every bucket exactly once with no partition on two ranks in a round;
a 2-rank epoch leaves every parameter bit-identical to a serial replay of the same lockstep
schedule (node updates on disjoint partitions; relation gradients summed g0 + g1, fp32 addition
being commutative), and the relation replicas bit-identical across ranks.
"""
import os
import socket
import sys

import numpy as np
import pytest

torch = pytest.importorskip("torch")

import paper_2101_08358_b200 as eb  # noqa: E402
from paper_2101_08358_b200 import distributed as ed  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


@pytest.mark.parametrize("p,world", [(2, 1), (4, 1), (4, 2), (8, 2), (8, 4), (16, 1), (16, 2), (16, 4), (16, 8),
                                     (32, 8), (1, 1)])
def test_round_schedule_is_conflict_free_cover(p, world):
    plan = ed.make_rounds(p, world)
    assert plan.rounds == max(1, p - 1)
    assert sorted(plan.order.tolist()) == list(range(p * p)), "every bucket exactly once"
    for r in range(plan.rounds):
        assert set(np.unique(plan.holder[r]).tolist()) == set(range(world))
        counts = []
        for g in range(world):
            held = set(plan.partitions(r, g))
            assert len(held) == p // world
            bk = plan.buckets(r, g)
            counts.append(len(bk))
            for _, i, j in bk:
                assert i in held and j in held, "bucket trained on a rank that does not hold its partitions"
        assert len(set(counts)) == 1, "rounds balanced across ranks (bucket count)"
    # self-buckets at first residency (round 0)
    for s in range(p * p):
        i, j = divmod(int(plan.order[s]), p)
        if i == j:
            assert plan.round[s] == 0
    # positions are grouped by round, then rank
    assert (np.diff(plan.round.astype(np.int64)) >= 0).all()


@pytest.mark.parametrize("p,world", [(4, 1), (8, 1), (8, 2), (16, 1), (16, 2), (16, 4), (32, 4), (32, 8), (64, 16)])
def test_overlapped_schedule_departing_pairs_first(p, world):
    """Coset schedule: a conflict-free cover like the circle method, and every partition that leaves
    its GPU after a round is used only by that GPU's early buckets, which come first in its round;
    each GPU receives exactly the pairs it sends (2 partitions per coset per round)."""
    plan = ed.make_rounds(p, world, overlap=True)
    assert plan.rounds == p - 1
    assert sorted(plan.order.tolist()) == list(range(p * p))
    for r in range(plan.rounds):
        for g in range(world):
            held = set(plan.partitions(r, g))
            assert len(held) == p // world
            sel = np.nonzero((plan.round == r) & (plan.rank == g))[0]
            flags = plan.early[sel]
            assert flags.tolist() == sorted(flags.tolist(), reverse=True), "early buckets first"
            for s_ in sel:
                i, j = divmod(int(plan.order[s_]), p)
                assert i in held and j in held
        if r + 1 < plan.rounds:
            for x, src, dst in plan.transfers(r):
                uses = [s_ for s_ in range(p * p) if plan.round[s_] == r and x in divmod(int(plan.order[s_]), p)]
                assert uses and all(plan.early[s_] for s_ in uses), "a departing partition trains early only"
            into = np.bincount([dst for _, _, dst in plan.transfers(r)], minlength=world)
            out = np.bincount([src for _, src, _ in plan.transfers(r)], minlength=world)
            assert (into == out).all() and into.max() <= 2 * (p // 4) // world


def test_round_schedule_handoff_volume():
    """p=16 over 8 GPUs: every round moves at most 2 partitions into each GPU (and the greedy
    assignment keeps at least one partition in place for most GPUs)."""
    plan = ed.make_rounds(16, 8)
    for r in range(plan.rounds - 1):
        moves = plan.transfers(r)
        into = np.bincount([dst for _, _, dst in moves], minlength=8)
        assert into.max() <= 2
        assert len(moves) <= 16


def test_round_schedule_errors():
    for p, w in [(3, 1), (4, 3), (16, 3), (1, 2), (0, 1)]:
        with pytest.raises(eb.ConfigError):
            ed.make_rounds(p, w)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


CFG = dict(kind="distmult", dim=16, V=1200, R=6, p=4, nt=32, alpha=0.5, neg_seed=3, b=150, seed=11, epochs=2)


def _graph():
    edges, split = eb.generate_graph(CFG["V"], CFG["R"], 4000, seed=5, train_frac=0.9, valid_frac=0.05)
    return eb.bucket_edges(edges[split == 0], CFG["V"], CFG["p"])


def _backend(edges):
    sys.path.insert(0, HERE)
    from dist_oracle_backend import OracleBackend
    return OracleBackend(CFG["kind"], CFG["dim"], CFG["V"], CFG["R"], CFG["p"], CFG["nt"], CFG["alpha"],
                         CFG["neg_seed"], edges)


def _worker(rank, world, port, out_dir, cfg=None):
    import torch.distributed as dist
    if cfg:
        CFG.update(cfg)
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    edges, off = _graph()
    be = _backend(edges)
    tr = ed.DistributedTrainer(be, CFG["p"], off, CFG["b"], rank, world, relations=CFG["kind"] != "dot", dist=dist,
                               overlap=CFG.get("overlap", False))
    tr.init_embeddings(CFG["seed"])
    n = 0
    for ep in range(CFG["epochs"]):
        n += tr.train_epoch(ep)["edges"]
    held = sorted(be.held)
    np.savez(os.path.join(out_dir, f"rank{rank}.npz"), held=np.array(held), theta=be.theta, acc=be.acc,
             rel_theta=be.rel_theta, rel_acc=be.rel_acc, edges=np.array([n]), hb=np.array([tr.handoff_bytes]),
             early=np.array([tr.report.early_handoffs]), handoffs=np.array([tr.report.handoffs]))
    dist.barrier()
    dist.destroy_process_group()


def _serial_replay(world):
    return _serial_replay_cfg(world)


def _serial_replay_cfg(world):
    """The same lockstep schedule in one process: all ranks' batches of a step, node updates in
    place, relation gradients summed in rank order before one relation Adagrad."""
    edges, off = _graph()
    be = _backend(edges)
    for x in range(CFG["p"]):
        be.init_partition(x, CFG["seed"])
    be.init_relations(CFG["seed"])
    plan = ed.make_rounds(CFG["p"], world, overlap=CFG.get("overlap", False))
    n = 0
    for ep in range(CFG["epochs"]):
        for r in range(plan.rounds):
            lists = [ed.round_batches(plan, off, CFG["b"], r, g) for g in range(world)]
            for s in range(max(len(x) for x in lists)):
                total = torch.zeros_like(be.rel_grad_t)
                for g in range(world):
                    if s < len(lists[g]):
                        pos, i, j, k, lo, hi, begin, nb = lists[g][s]
                        be.train_batch(pos, i, j, k, lo, hi, begin, nb, ep)
                        total = total + be.rel_grad_t  # fp32, rank order
                        n += nb
                be.rel_grad_t.copy_(total)
                be.apply_relations()
    return be, n, off


def test_two_rank_epochs_bit_identical_to_serial_replay(tmp_path):
    import torch.multiprocessing as mp
    world = 2
    port = _free_port()
    mp.start_processes(_worker, args=(world, port, str(tmp_path)), nprocs=world, join=True, start_method="spawn")
    ref, n_ref, off = _serial_replay(world)
    assert n_ref == CFG["epochs"] * int(off[-1])
    got_theta = np.full_like(ref.theta, np.nan)
    got_acc = np.full_like(ref.acc, np.nan)
    total_edges = 0
    rel = []
    for g in range(world):
        z = np.load(tmp_path / f"rank{g}.npz")
        total_edges += int(z["edges"][0])
        for x in z["held"]:
            o, sz = eb.partition_offset(CFG["V"], CFG["p"], int(x)), eb.partition_size(CFG["V"], CFG["p"], int(x))
            got_theta[o:o + sz] = z["theta"][o:o + sz]
            got_acc[o:o + sz] = z["acc"][o:o + sz]
        rel.append((z["rel_theta"], z["rel_acc"]))
        assert int(z["hb"][0]) > 0, "partitions were handed off between rounds"
    assert total_edges == n_ref, "every training edge consumed exactly once per epoch"
    assert not np.isnan(got_theta).any(), "every partition ends on exactly one rank"
    assert got_theta.tobytes() == ref.theta.tobytes()
    assert got_acc.tobytes() == ref.acc.tobytes()
    assert rel[0][0].tobytes() == rel[1][0].tobytes() == ref.rel_theta.tobytes(), "relation replicas identical"
    assert rel[0][1].tobytes() == rel[1][1].tobytes() == ref.rel_acc.tobytes()


@pytest.mark.gpu
@pytest.mark.parametrize("kind", ["complex", "dot"])
def test_gpu_backend_single_rank_matches_direct_training(kind):
    """The product backend (GpuBackend: C-ABI step, external relation reduction through an NCCL
    all-reduce on the context stream, dense relation Adagrad) on a 1-rank NCCL group leaves every
    parameter bit-identical to training the same bucket sequence directly (in-place relations)."""
    import torch.distributed as dist
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    V, R, p, d = 3000, 12, 4, 32
    edges, split = eb.generate_graph(V, R, 20000, seed=5, train_frac=0.9, valid_frac=0.05)
    bucketed, off = eb.bucket_edges(edges[split == 0], V, p)
    dev_edges = torch.from_numpy(bucketed.view(np.int32)).cuda()
    h = eb.Hyper(kind=kind, dim=d, batch_size=300, num_negatives=64, neg_seed=3, engine="tc")
    port = _free_port()
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1,
                            device_id=torch.device("cuda:0"))
    try:
        tr = eb.Trainer(h, V, R, p, device=0, allocate=False)
        be = ed.GpuBackend(tr, dev_edges)
        D = ed.DistributedTrainer(be, p, off, 300, 0, 1, relations=kind != "dot", dist=dist)
        D.init_embeddings(11)
        for ep in range(2):
            D.train_epoch(ep)
        torch.cuda.synchronize()
        ref = eb.Trainer(h, V, R, p, device=0)
        ref.init_embeddings(11)
        seq = np.stack([D.plan.order // p, D.plan.order % p], 1)
        for ep in range(2):
            ref.train_epoch(dev_edges, off, seq, ep)
        th_ref, ac_ref = ref.node_table()
        tabs = D.local_tables()
        th = eb.rows_to_disk(np.concatenate([tabs[x][0].cpu().numpy() for x in range(p)]), kind)
        ac = eb.rows_to_disk(np.concatenate([tabs[x][1].cpu().numpy() for x in range(p)]), kind)
        assert th.tobytes() == th_ref.tobytes()
        assert ac.tobytes() == ac_ref.tobytes()
        if kind != "dot":
            assert tr.rel_theta.cpu().numpy().tobytes() == ref.rel_theta.cpu().numpy().tobytes()
            assert tr.rel_acc.cpu().numpy().tobytes() == ref.rel_acc.cpu().numpy().tobytes()
    finally:
        dist.destroy_process_group()


GCFG = dict(kind="complex", dim=32, V=3000, R=12, p=4, b=300, nt=64, seed=11, epochs=2)


def _gpu_graph():
    edges, split = eb.generate_graph(GCFG["V"], GCFG["R"], 20000, seed=5, train_frac=0.9, valid_frac=0.05)
    return eb.bucket_edges(edges[split == 0], GCFG["V"], GCFG["p"])


def _gpu_hyper():
    return eb.Hyper(kind=GCFG["kind"], dim=GCFG["dim"], batch_size=GCFG["b"], num_negatives=GCFG["nt"], neg_seed=3,
                    engine="tc")


def _gpu_worker(rank, world, port, out_dir):
    import torch.distributed as dist
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    bucketed, off = _gpu_graph()
    dev = torch.from_numpy(bucketed.view(np.int32)).cuda()
    tr = eb.Trainer(_gpu_hyper(), GCFG["V"], GCFG["R"], GCFG["p"], device=0, allocate=False)
    D = ed.DistributedTrainer(ed.GpuBackend(tr, dev), GCFG["p"], off, GCFG["b"], rank, world, relations=True,
                              dist=dist)
    D.init_embeddings(GCFG["seed"])
    for ep in range(GCFG["epochs"]):
        D.train_epoch(ep)
    torch.cuda.synchronize()
    k = GCFG["kind"]
    tabs = {x: (eb.rows_to_disk(t[0].cpu().numpy(), k), eb.rows_to_disk(t[1].cpu().numpy(), k))
            for x, t in D.local_tables().items()}
    np.savez(os.path.join(out_dir, f"g{rank}.npz"), held=np.array(sorted(tabs)),
             **{f"th{x}": v[0] for x, v in tabs.items()}, **{f"ac{x}": v[1] for x, v in tabs.items()},
             rel_theta=tr.relation_table()[0], rel_acc=tr.relation_table()[1])
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.gpu
def test_gpu_two_rank_epochs_bit_identical_to_serial_replay(tmp_path):
    """Two processes on one GPU run the product backend (C-ABI steps, external relation gradients,
    partition handoffs) over gloo; every parameter equals a serial replay of the same lockstep
    schedule on one context (both ranks' batches of a step, relation gradients summed g0 + g1 before
    one dense relation Adagrad)."""
    import torch.multiprocessing as mp
    import paper_2101_08358_b200._lib as L
    world, port = 2, _free_port()
    mp.start_processes(_gpu_worker, args=(world, port, str(tmp_path)), nprocs=world, join=True, start_method="spawn")
    # serial replay on one context
    bucketed, off = _gpu_graph()
    dev = torch.from_numpy(bucketed.view(np.int32)).cuda()
    tr = eb.Trainer(_gpu_hyper(), GCFG["V"], GCFG["R"], GCFG["p"], device=0)
    tr.init_embeddings(GCFG["seed"])
    g = [torch.zeros((GCFG["R"], GCFG["dim"]), device="cuda") for _ in range(world)]
    plan = ed.make_rounds(GCFG["p"], world)
    base = dev.data_ptr()
    for ep in range(GCFG["epochs"]):
        for r in range(plan.rounds):
            lists = [ed.round_batches(plan, off, GCFG["b"], r, k) for k in range(world)]
            for s_ in range(max(len(x) for x in lists)):
                for k in range(world):
                    L.check(L.lib().ember_relations_external(tr.ctx, g[k].data_ptr()))
                    if s_ < len(lists[k]):
                        pos, i, j, kk, lo, hi, begin, nb = lists[k][s_]
                        L.check(L.lib().ember_train_batch(tr.ctx, base + 12 * lo, hi - lo, begin, nb, i, j, ep, pos, kk,
                                                          None))
                    else:
                        with torch.cuda.stream(tr.torch_stream()):
                            g[k].zero_()
                with torch.cuda.stream(tr.torch_stream()):
                    total = g[0] + g[1]
                L.check(L.lib().ember_relations_apply_dense(tr.ctx, total.data_ptr()))
                tr.torch_stream().synchronize()
    L.check(L.lib().ember_relations_external(tr.ctx, None))
    th, ac = tr.node_table()
    rt, ra = tr.relation_table()
    seen = set()
    for k in range(world):
        z = np.load(tmp_path / f"g{k}.npz")
        assert z["rel_theta"].tobytes() == rt.tobytes() and z["rel_acc"].tobytes() == ra.tobytes()
        for x in z["held"]:
            o, n = eb.partition_offset(GCFG["V"], GCFG["p"], int(x)), eb.partition_size(GCFG["V"], GCFG["p"], int(x))
            assert z[f"th{x}"].tobytes() == th[o:o + n].tobytes(), f"partition {x}"
            assert z[f"ac{x}"].tobytes() == ac[o:o + n].tobytes()
            seen.add(int(x))
    assert seen == set(range(GCFG["p"]))


def test_seek_transfers_reach_the_round_layout():
    plan = ed.make_rounds(16, 8)
    for r in range(plan.rounds):
        held = plan.holder[0].copy()
        for x, src, dst in plan.transfers(0, r):
            assert held[x] == src
            held[x] = dst
        assert (held == plan.holder[r]).all()


def test_two_rank_overlapped_schedule_bit_identical_to_serial_replay(tmp_path):
    """The coset schedule (p=8 over 2 ranks) through the library's round loop: handoffs issued after
    the departing pairs' buckets, mid-round, and every parameter still equals the serial replay."""
    import torch.multiprocessing as mp
    world, port = 2, _free_port()
    cfg = dict(p=8, V=1600, epochs=2, overlap=True)
    saved = dict(CFG)
    try:
        CFG.update(cfg)
        mp.start_processes(_worker, args=(world, port, str(tmp_path), cfg), nprocs=world, join=True,
                           start_method="spawn")
        ref, n_ref, off = _serial_replay(world)
        got = np.full_like(ref.theta, np.nan)
        total, early, hand = 0, 0, 0
        rel = []
        for g in range(world):
            z = np.load(tmp_path / f"rank{g}.npz")
            total += int(z["edges"][0])
            early += int(z["early"][0])
            hand += int(z["handoffs"][0])
            rel.append(z["rel_theta"])
            for x in z["held"]:
                o, sz = eb.partition_offset(CFG["V"], CFG["p"], int(x)), eb.partition_size(CFG["V"], CFG["p"], int(x))
                got[o:o + sz] = z["theta"][o:o + sz]
        assert total == n_ref
        assert got.tobytes() == ref.theta.tobytes()
        assert rel[0].tobytes() == rel[1].tobytes() == ref.rel_theta.tobytes()
        assert hand > 0 and early > 0, "handoffs issued before the end of their round"
    finally:
        CFG.clear()
        CFG.update(saved)


def test_four_rank_dot_epochs_bit_identical_to_serial_replay(tmp_path):
    """Dot model (no relations, no per-step collective) over 4 ranks, p=8: the handoffs alone must
    reproduce the serial replay bit for bit."""
    import torch.multiprocessing as mp
    world, port = 4, _free_port()
    cfg = dict(kind="dot", p=8, V=1600, epochs=2)
    saved = dict(CFG)
    try:
        CFG.update(cfg)
        mp.start_processes(_worker, args=(world, port, str(tmp_path), cfg), nprocs=world, join=True,
                           start_method="spawn")
        ref, n_ref, off = _serial_replay(world)
        got = np.full_like(ref.theta, np.nan)
        total = 0
        for g in range(world):
            z = np.load(tmp_path / f"rank{g}.npz")
            total += int(z["edges"][0])
            for x in z["held"]:
                o, sz = eb.partition_offset(CFG["V"], CFG["p"], int(x)), eb.partition_size(CFG["V"], CFG["p"], int(x))
                got[o:o + sz] = z["theta"][o:o + sz]
        assert total == n_ref
        assert got.tobytes() == ref.theta.tobytes()
    finally:
        CFG.clear()
        CFG.update(saved)


@pytest.mark.gpu
@pytest.mark.parametrize("kind,overlap", [("complex", True), ("complex", False), ("dot", True)])
def test_native_driver_single_rank_matches_direct_training(kind, overlap):
    """The all-native multi-GPU driver (ember_dist_*: C++ round loop, driver-owned partition slots,
    NCCL paths idle at world 1) at world 1: two epochs leave every parameter bit-identical to the
    same buckets trained through ember_train_epoch in schedule order."""
    p, V, R = 4, 3000, 12
    edges, split = eb.generate_graph(V, R, 20000, seed=5, train_frac=0.9, valid_frac=0.05)
    bucketed, off = eb.bucket_edges(edges[split == 0], V, p)
    dev = torch.from_numpy(bucketed.view(np.int32)).cuda()
    h = eb.Hyper(kind=kind, dim=32, batch_size=300, num_negatives=64, neg_seed=3, engine="tc")
    tr = eb.Trainer(h, V, R, p, device=0, allocate=False)
    D = ed.NativeDistributed(tr, dev, off, 0, 1, overlap=overlap)
    D.init_embeddings(11)
    for ep in range(2):
        rep = D.train_epoch(ep)
        assert rep.edges == int(off[-1]) and rep.moved_partitions == 0
    assert np.isfinite(D.loss())
    got = {x: D.partition_table(x) for x in D.held()}
    assert sorted(got) == list(range(p))
    rel = tr.relation_table() if kind != "dot" else None
    D.close()
    ref = eb.Trainer(h, V, R, p, device=0)
    ref.init_embeddings(11)
    seq = np.stack([D.plan.order // p, D.plan.order % p], 1)
    for ep in range(2):
        ref.train_epoch(dev, off, seq, ep)
    th_ref, ac_ref = ref.node_table()
    for x in range(p):
        o, n = eb.partition_offset(V, p, x), eb.partition_size(V, p, x)
        assert got[x][0].tobytes() == th_ref[o:o + n].tobytes(), f"partition {x}"
        assert got[x][1].tobytes() == ac_ref[o:o + n].tobytes()
    if rel is not None:
        assert rel[0].tobytes() == ref.relation_table()[0].tobytes()
    tr.close()
    ref.close()
