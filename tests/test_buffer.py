"""Device partition buffer through the C-ABI.

SPEC invariants checked here:
  * replaying a plan yields exactly plan.swap_count misses after the initial c loads, and the
    buffer's eviction decisions equal the reference ordering's Belady trace (ordering.cpp
    :94-159, restated bit-identically in csrc/host/ordering.cpp and pinned by test_ordering.py);
  * no lost updates: an epoch through the buffer leaves every parameter bit-identical to the
    same epoch with all partitions resident (same bucket sequence, same update stream);
  * IO counters: reads = writes = c + swap_count per epoch (simulate_io);
  * memory ceiling: c + 2 device slots.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2101_08358_b200 as eb  # noqa: E402

from gpu_helpers import make_graph  # noqa: E402


def _trainers(kind, dim, V, R, p, engine, b=256, nt=64):
    h = eb.Hyper(kind=kind, dim=dim, batch_size=b, num_negatives=nt, neg_seed=3, engine=engine)
    resident = eb.Trainer(h, V, R, p, device=0)
    resident.init_embeddings(11)
    buffered = eb.Trainer(h, V, R, p, device=0, allocate=False)
    return resident, buffered


@pytest.mark.parametrize("kind,engine,order,p,c,seed", [
    ("complex", "tc", "elimination", 4, 2, 42),
    ("distmult", "tc", "random", 6, 3, 7),
    ("dot", "simt", "hilbert", 4, 2, 0),
    ("complex", "tc", "elimination", 5, 5, 1),   # c == p: no swaps, no staging slots
])
def test_buffered_epochs_bit_identical_to_resident(kind, engine, order, p, c, seed):
    V, R = 4000, 16
    edges, off, _ = make_graph(V=V, R=R, E=30000, p=p, seed=9)
    dev_edges = torch.from_numpy(edges.view(np.int32)).cuda()
    plan = eb.make_plan(order, p, c, seed)
    resident, buffered = _trainers(kind, 32, V, R, p, engine)
    buf = eb.PartitionBuffer(buffered, c, plan["seq"])
    buf.init_backing(11)

    # decisions == the ordering module's Belady trace
    dec = buf.decisions()
    assert len(dec) == plan["swap_count"]
    if plan["swap_count"]:
        assert (dec == np.asarray(plan["swaps"]).reshape(-1, 3)).all()

    epochs = 2
    for ep in range(epochs):
        a = resident.train_epoch(dev_edges, off, plan["seq"], ep)
        b = buf.train_epoch(dev_edges, off, ep)
        assert a["batches"] == b["batches"] and a["edges"] == b["edges"] == int(off[-1])
        assert a["loss"] == pytest.approx(b["loss"], rel=1e-12)
    th_r, ac_r = resident.node_table()
    th_b, ac_b = buf.node_table()
    assert th_r.tobytes() == th_b.tobytes(), "lost or misplaced updates through the buffer"
    assert ac_r.tobytes() == ac_b.tobytes()
    if resident.rel_theta is not None:
        assert resident.rel_theta.cpu().numpy().tobytes() == buffered.rel_theta.cpu().numpy().tobytes()

    st = buf.stats()
    fills = min(c, p)
    assert st["swaps_per_epoch"] == plan["swap_count"]
    assert st["epochs"] == epochs
    assert st["reads"] == epochs * (fills + plan["swap_count"])
    assert st["writes"] == epochs * (fills + plan["swap_count"])
    assert st["slots"] == c + (2 if c < p else 0)
    assert st["stall_ms"] >= 0.0
    buf.close()
    resident.close()
    buffered.close()


def test_fig7_five_misses_and_order_errors():
    """PAPER Fig. 7 / SPEC.md:312: the elimination plan p=4, c=2 has exactly five misses."""
    V, R, p, c = 4000, 16, 4, 2
    edges, off, _ = make_graph(V=V, R=R, E=8000, p=p, seed=9)
    plan = eb.make_plan("elimination", p, c, 42)
    _, tr = _trainers("distmult", 16, V, R, p, "tc")
    buf = eb.PartitionBuffer(tr, c, plan["seq"])
    buf.init_backing(11)
    assert len(buf.decisions()) == 5
    with pytest.raises(eb.ConfigError):
        buf.acquire(1)  # an epoch starts at step 0
    assert buf.acquire(0) == tuple(int(x) for x in plan["seq"][0])
    with pytest.raises(eb.ConfigError):
        buf.acquire(2)  # plan order
    buf.release(0)
    with pytest.raises(eb.ConfigError):
        eb.PartitionBuffer(tr, 1, plan["seq"])  # c >= 2 when p > 1
    bad = np.array(plan["seq"]).copy()
    bad[2:4] = bad[0:2]
    with pytest.raises(eb.ConfigError):
        eb.PartitionBuffer(tr, c, bad)  # not a permutation of the buckets


def test_checkpoint_files_feed_the_buffer(tmp_path):
    """save_trainer writes the graph store's node_part_<k>.bin / relations.bin;
    a buffer whose backing store is loaded from them trains bit-identically to the resident run,
    and the backing store written back after the epoch equals the resident tables."""
    from paper_2101_08358_b200 import storage
    V, R, p, c = 4000, 16, 4, 2
    edges, off, _ = make_graph(V=V, R=R, E=20000, p=p, seed=9)
    dev = torch.from_numpy(edges.view(np.int32)).cuda()
    plan = eb.make_plan("elimination", p, c, 42)
    resident, buffered = _trainers("complex", 32, V, R, p, "tc")
    storage.save_trainer(str(tmp_path / "ck0"), resident)
    fresh = eb.Trainer(resident.h, V, R, p, device=0)
    storage.load_trainer(str(tmp_path / "ck0"), fresh)
    assert fresh.node_table()[0].tobytes() == resident.node_table()[0].tobytes()
    buf = eb.PartitionBuffer(buffered, c, plan["seq"])
    storage.load_buffer_backing(str(tmp_path / "ck0"), buf)
    buffered.rel_theta.copy_(resident.rel_theta)
    buffered.rel_acc.copy_(resident.rel_acc)
    resident.train_epoch(dev, off, plan["seq"], 0)
    buf.train_epoch(dev, off, 0)
    storage.save_buffer_backing(str(tmp_path / "ck1"), buf)
    th, ac = resident.node_table()
    for k in range(p):
        o, n = eb.partition_offset(V, p, k), eb.partition_size(V, p, k)
        t2, a2 = storage.read_node_part(str(tmp_path / "ck1"), k, n, 32)
        assert t2.tobytes() == th[o:o + n].tobytes() and a2.tobytes() == ac[o:o + n].tobytes()
