"""bench.py's output contract on the CPU-only arm: `--impl reference` prints exactly one JSON line
on stdout (native chatter goes to stderr) carrying the keys the driver reads."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_prints_one_json_line():
    r = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--steps", "1", "--warmup", "3",
                        "--config", "fb15k237"], cwd=ROOT, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.strip()]
    assert len(lines) == 1, r.stdout
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "impl",
              "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["impl"] == "reference" and d["value"] > 0
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["cpu_baseline"]["kind"] == "port"
    # the reference arm runs the CPU restatement only: no product library in the process
    assert d["native_libraries"] and all(x.startswith("oracle/") for x in d["native_libraries"]), d["native_libraries"]
    assert "paper_2101_08358_b200" not in r.stderr
    # same batch stream as the GPU arm: full batches from its timed window
    assert d["config"]["batch"] == 10_000 and d["config"]["first_batch"] == 27 // 3 + 3
