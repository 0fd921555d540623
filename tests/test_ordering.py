"""BETA / bucket-order parity: our ordering (paper_2101_08358_b200/csrc/host/ordering.cpp via the
C-ABI) must be bit-identical to the reference's ordering.cpp — against committed golden plans
(tests/golden/reference_rng_ordering.json, produced by oracle/_ref) and, when the reference build
is present, live against oracle/_ref for a sweep of (kind, p, c, seed)."""
import json
import os
import subprocess

import numpy as np
import pytest

import paper_2101_08358_b200 as eb

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "reference_rng_ordering.json")))
REF_DIR = os.path.join(os.path.dirname(os.path.dirname(__file__)), "oracle", "_ref")


def _ref():
    from oracle import pyoracle as po
    if not os.path.exists(os.path.join(REF_DIR, "libember_ref.so")):
        if os.path.isdir("/root/reference/proj"):
            po.build(ref=True)
        else:
            return None
    return po


@pytest.mark.parametrize("case", GOLD["plans"], ids=lambda c: f"k{c['kind']}-p{c['p']}-c{c['c']}-s{c['seed']}")
def test_plans_match_reference_golden(case):
    plan = eb.make_plan(case["kind"], case["p"], case["c"], case["seed"])
    assert plan["seq"].reshape(-1).tolist() == case["seq"]
    assert plan["swap_count"] == case["swap_count"]
    assert plan["admissions"].tolist() == case["admissions"]
    assert plan["swaps"].reshape(-1).tolist() == case["swaps"]
    assert plan["bucket_state"].tolist() == case["bucket_state"]


def test_paper_figure_counts():
    assert eb.make_plan("elimination", 4, 2, 42)["swap_count"] == 5   # Fig. 7
    assert eb.make_plan("hilbert", 4, 2, 0)["swap_count"] == 9        # Fig. 7
    assert eb.make_plan("elimination", 6, 3, 7)["swap_count"] == 7
    assert eb.lower_bound_swaps(6, 3) == 6 and eb.lower_bound_swaps(128, 32) == 247
    p16 = eb.make_plan("elimination", 16, 16, 0)
    assert p16["swap_count"] == 0
    assert p16["seq"].tolist() == [[i, j] for i in range(16) for j in range(16)]  # p == c: lexicographic


def test_formula_equals_construction_exhaustive():
    for p in range(2, 65):
        for c in range(2, p + 1):
            assert eb.make_plan("elimination", p, c, 1000 * p + c)["swap_count"] == eb.elimination_swap_formula(p, c)


def test_config_errors():
    with pytest.raises(eb.ConfigError):
        eb.make_plan("elimination", 3, 1, 0)
    with pytest.raises(eb.ConfigError):
        eb.make_plan("elimination", 3, 4, 0)
    with pytest.raises(eb.ConfigError):
        eb.lower_bound_swaps(4, 1)


def test_live_against_reference_build():
    po = _ref()
    if po is None or po.ref_lib() is None:
        pytest.skip("oracle/_ref not built and /root/reference absent")
    rng = np.random.default_rng(0)
    for _ in range(300):
        kind = int(rng.integers(0, 4))
        p = int(rng.integers(1, 40))
        c = int(rng.integers(1 if p == 1 else 2, p + 1))
        seed = int(rng.integers(0, 2**63))
        ours = eb.make_plan(kind, p, c, seed)
        ref = po.ref_plan(kind, p, c, seed)
        assert (ours["seq"] == ref["seq"]).all(), (kind, p, c, seed)
        assert ours["swap_count"] == ref["swap_count"]
        assert (ours["admissions"] == ref["admissions"]).all()
        assert (ours["swaps"] == ref["swaps"]).all()
        assert (ours["bucket_state"] == ref["bucket_state"]).all()


def test_reference_unit_test_passes_in_place():
    exe = os.path.join(REF_DIR, "test_ordering")
    if not os.path.exists(exe):
        if not os.path.isdir("/root/reference/proj"):
            pytest.skip("reference test binary not built here")
        _ref().build(ref=True)
    out = subprocess.run([exe], capture_output=True, text=True, timeout=120)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "16 passed" in out.stdout


_VALIDATE_CPP = r"""
#include "ember/ordering.h"
#include <cstdio>
#include <functional>
using namespace ember;
static int rejects(const std::function<void(OrderingPlan&)>& corrupt, const OrderingPlan& good) {
    OrderingPlan bad = good;
    corrupt(bad);
    try { bad.validate(); } catch (const EmberError&) { return 0; }
    return 1;
}
int main() {
    int fails = 0;
    for (auto kind : {OrderingKind::Elimination, OrderingKind::Hilbert, OrderingKind::HilbertSymmetric,
                      OrderingKind::Random})
        for (unsigned p : {1u, 4u, 7u, 16u})
            for (unsigned c : {2u, 3u, 5u}) {
                if (c > p) continue;
                OrderingPlan plan = make_plan(kind, p, c, 42);
                plan.validate();  // every generated plan is valid
                if (plan.swap_events.empty()) continue;
                fails += rejects([](OrderingPlan& q) { q.bucket_sequence.pop_back(); }, plan);
                fails += rejects([](OrderingPlan& q) { q.bucket_sequence[1] = q.bucket_sequence[0]; }, plan);
                fails += rejects([](OrderingPlan& q) { q.swap_count += 1; }, plan);
                fails += rejects([](OrderingPlan& q) { std::swap(q.swap_events[0].evicted, q.swap_events[0].admitted); }, plan);
                fails += rejects([](OrderingPlan& q) { q.bucket_state.back() = 0; }, plan);
                fails += rejects([](OrderingPlan& q) { q.buffer_states[1].push_back(q.p); }, plan);
            }
    try { make_plan(OrderingKind::Elimination, 4, 5, 0); ++fails; } catch (const ConfigError&) {}
    try { make_plan(OrderingKind::Elimination, 4, 1, 0); ++fails; } catch (const ConfigError&) {}
    std::printf("validate fails=%d\n", fails);
    return fails != 0;
}
"""


def test_plan_validation_accepts_generated_and_rejects_corrupted_plans(tmp_path):
    """OrderingPlan::validate (ordering.h:45) accepts every generated plan and throws EmberError for
    each structural corruption; bad (p, c) raise ConfigError."""
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    src = tmp_path / "validate.cpp"
    src.write_text(_VALIDATE_CPP)
    exe = tmp_path / "validate"
    subprocess.run(["g++", "-std=c++20", "-O1", "-I", os.path.join(root, "include"), str(src),
                    os.path.join(root, "paper_2101_08358_b200", "csrc", "host", "ordering.cpp"), "-o", str(exe)],
                   check=True)
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0 and "fails=0" in r.stdout, r.stdout + r.stderr
