"""The step's hand-written (key, slot) sort (csrc/sort.cu) through ember_debug_sort_slots, bit-exact
against numpy's stable argsort and run-length encoding: sorted keys and slots, rank (inverse
permutation), run keys / offsets / count and the unique-slot flags. Shapes: the FB86m bench's
152 k slots with power-law hot keys (24-bit keys), ragged tile tails, 1-4 radix passes, all-equal
keys, every key distinct, and the context's full slot capacity."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from gpu_helpers import make_trainer  # noqa: E402


@pytest.fixture(scope="module")
def trainer():
    # cap_rows = 3 * 50000 + 2 * 1000 = 152,000 gradient slots (the bench's batch geometry)
    return make_trainer("complex", dim=16, b=50000, nt=1000, V=3000, engine="tc")


def _expect(keys):
    order = np.argsort(keys, kind="stable").astype(np.uint32)
    ks = keys[order]
    head = np.ones(len(ks), bool)
    head[1:] = ks[1:] != ks[:-1]
    starts = np.flatnonzero(head).astype(np.uint32)
    counts = np.diff(np.append(starts, len(ks)))
    rank = np.empty(len(ks), np.uint32)
    rank[order] = np.arange(len(ks), dtype=np.uint32)
    uniq_sorted = np.repeat(counts == 1, counts)
    uniq = np.empty(len(ks), np.uint8)
    uniq[order] = uniq_sorted
    return order, ks, rank, uniq, ks[starts], np.append(starts, len(ks)).astype(np.uint32)


def _check(tr, keys, bits):
    keys = np.ascontiguousarray(keys, dtype=np.uint32)
    got = tr.debug_sort_slots(torch.from_numpy(keys.view(np.int32)).cuda(), bits)
    order, ks, rank, uniq, ukeys, offsets = _expect(keys)
    nr = int(got["nruns"][0])
    assert nr == len(ukeys)
    assert (got["keys_sorted"] == ks).all()
    assert (got["vals_sorted"] == order).all()
    assert (got["rank"] == rank).all()
    assert (got["uniq"] == uniq).all()
    assert (got["ukeys"][:nr] == ukeys).all()
    assert (got["offsets"][: nr + 1] == offsets).all()


def _power_law_keys(rng, n, hi, a=1.2):
    z = rng.zipf(a, size=n).astype(np.uint64) - 1
    return ((z * 2654435761) % hi).astype(np.uint32)


def test_sort_bench_shape_hot_keys(trainer):
    rng = np.random.default_rng(1)
    nb, n_neg, node_range = 50000, 2000, 10_757_000
    nodes = _power_law_keys(rng, 2 * nb + n_neg, node_range)
    rels = node_range + _power_law_keys(rng, nb, 14824, a=1.5)
    _check(trainer, np.concatenate([nodes, rels]), 24)


@pytest.mark.parametrize("n", [1, 31, 33, 4095, 4096, 4097, 12289, 100003])
@pytest.mark.parametrize("bits", [8, 13, 24, 32])
def test_sort_ragged_sizes_and_passes(trainer, n, bits):
    rng = np.random.default_rng(n * 37 + bits)
    hi = (1 << bits) - 1
    keys = rng.integers(0, min(hi, 4 * n) + 1, size=n, dtype=np.uint64).astype(np.uint32)
    if bits == 32 and n > 4:
        keys[:3] = [0xFFFFFFFF, 0, 0x80000000]
    _check(trainer, keys, bits)


def test_sort_all_equal_and_all_distinct(trainer):
    n = 152000
    _check(trainer, np.full(n, 7, np.uint32), 24)
    _check(trainer, np.random.default_rng(3).permutation(n).astype(np.uint32), 24)
    _check(trainer, np.arange(n, dtype=np.uint32)[::-1].copy(), 18)


def test_sort_rejects_oversize(trainer):
    import paper_2101_08358_b200 as eb

    keys = torch.zeros(152001, dtype=torch.int32, device="cuda")
    with pytest.raises(eb.EmberError):
        trainer.debug_sort_slots(keys, 24)
