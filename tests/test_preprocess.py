"""Graph-store preprocessing (ingest, partition_nodes, bucket_edges).

CPU: the oracle's restatement against SPEC's examples and invariants (dense ids, uniform
contiguous partitions, a seeded shuffle that is a permutation, determinism, bucketing as a
partition of the train split). GPU: ember_graph_preprocess bit-identical to the oracle."""
import numpy as np
import pytest

from oracle import pyoracle as po


def _raw(n=5000, seed=0):
    rng = np.random.default_rng(seed)
    toks = rng.choice(2**31, size=700, replace=False).astype(np.uint32)  # sparse node tokens
    rels = rng.choice(2**20, size=9, replace=False).astype(np.uint32)
    return np.stack([rng.choice(toks, n), rng.choice(rels, n), rng.choice(toks, n)], 1).astype(np.uint32)


def test_spec_counting_example():
    # "a r1 b / b r1 c / a r2 c", split (1,0,0) -> |V|=3, |R|=2, |E|=3
    a, b, c, r1, r2 = 10, 20, 30, 7, 9
    out = po.preprocess(np.array([[a, r1, b], [b, r1, c], [a, r2, c]]), 1, 5, 1.0, 0.0)
    assert out["num_nodes"] == 3 and out["num_relations"] == 2 and len(out["train"]) == 3
    assert sorted(out["node_tokens"].tolist()) == [a, b, c] and out["rel_tokens"].tolist() == [r1, r2]


def test_invariants_and_determinism():
    raw = _raw()
    p = 4
    o1 = po.preprocess(raw, p, 11, 0.8, 0.1)
    o2 = po.preprocess(raw, p, 11, 0.8, 0.1)
    for k in ("train", "valid", "test", "offsets", "node_tokens"):
        assert (o1[k] == o2[k]).all()
    V = o1["num_nodes"]
    n = len(raw)
    assert len(o1["train"]) == int(0.8 * n) and len(o1["valid"]) == int(0.1 * n)
    # relabeled edges map back to the raw multiset
    tok = o1["node_tokens"]
    rt = o1["rel_tokens"]
    back = np.concatenate([o1["train"], o1["valid"], o1["test"]])
    back = np.stack([tok[back[:, 0]], rt[back[:, 1]], tok[back[:, 2]]], 1)
    assert sorted(map(tuple, back.tolist())) == sorted(map(tuple, raw.tolist()))
    # buckets: edge (s, r, d) in bucket (part(s), part(d)), offsets cover the train split
    off = o1["offsets"].astype(np.int64)
    assert off[0] == 0 and off[-1] == len(o1["train"]) and (np.diff(off) >= 0).all()
    q, r = divmod(V, p)
    part = lambda x: np.where(x < r * (q + 1), x // (q + 1), r + (x - r * (q + 1)) // max(q, 1))  # noqa: E731
    for b in range(p * p):
        e = o1["train"][off[b]:off[b + 1]]
        assert (part(e[:, 0]) * p + part(e[:, 2]) == b).all()
    # the seeded permutation spreads tokens over partitions (not the sorted-token order)
    assert not (np.diff(tok.astype(np.int64)) > 0).all()
    o3 = po.preprocess(raw, p, 12, 0.8, 0.1)
    assert not (o3["node_tokens"] == tok).all()


@pytest.mark.gpu
@pytest.mark.parametrize("p,seed,tr,va", [(1, 3, 0.9, 0.05), (4, 11, 0.8, 0.1), (16, 5, 1.0, 0.0)])
def test_device_preprocessing_bit_identical_to_oracle(p, seed, tr, va):
    import paper_2101_08358_b200 as eb
    raw = _raw(20000, seed)
    got = eb.preprocess_graph(raw, p, seed, tr, va, device=0)
    exp = po.preprocess(raw, p, seed, tr, va)
    assert got["num_nodes"] == exp["num_nodes"] and got["num_relations"] == exp["num_relations"]
    assert (got["offsets"] == exp["offsets"]).all()
    for k in ("train", "valid", "test", "node_tokens", "rel_tokens"):
        g = got[k].cpu().numpy().view(np.uint32)
        assert g.shape == exp[k].shape and (g == exp[k]).all(), k
