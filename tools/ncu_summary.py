#!/usr/bin/env python
"""Summarises ncu output brought back in gpurun_out/ into committed profiles/ files.

  python tools/ncu_summary.py launches <launches.csv> <out.md>
      per-kernel launch count, summed device time and share of the timed region
      (ncu --metrics gpu__time_duration.sum --profile-from-start off over bench.py's timed steps)
  python tools/ncu_summary.py full <report.ncu-rep> <out.md> [algorithmic_bytes] [algorithmic_flops]
      the roofline-relevant metrics of a `ncu --set full` capture (one launch per kernel)
"""
from __future__ import annotations

import collections
import csv
import io
import re
import subprocess
import sys


def short(name: str) -> str:
    name = re.sub(r"\(.*", "", name)
    return name.replace("ember::<unnamed>::", "").replace("ember::", "")


def launches(path: str, out: str) -> None:
    text = open(path).read()
    rows = list(csv.reader(io.StringIO(text[text.index('"ID"'):])))
    h = rows[0]
    ki, mi, vi = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
    tot = collections.OrderedDict()
    for r in rows[1:]:
        if len(r) <= vi or r[mi] != "gpu__time_duration.sum":
            continue
        k = short(r[ki])
        c, t = tot.get(k, (0, 0.0))
        tot[k] = (c + 1, t + float(r[vi].replace(",", "")))
    all_ns = sum(t for _, t in tot.values())
    lines = [f"# Launch list: `{path.split('/')[-1]}`", "",
             "ncu `--metrics gpu__time_duration.sum --clock-control none --profile-from-start off` over bench.py's "
             "timed steps (cold-cache, serialised: compare shares, not absolutes).", "",
             "| kernel | launches | total µs | mean µs | share |", "|---|---:|---:|---:|---:|"]
    for k, (c, t) in sorted(tot.items(), key=lambda kv: -kv[1][1]):
        lines.append(f"| `{k}` | {c} | {t / 1e3:.1f} | {t / c / 1e3:.2f} | {100 * t / all_ns:.1f}% |")
    lines.append(f"| **total** | {sum(c for c, _ in tot.values())} | {all_ns / 1e3:.1f} | | 100% |")
    open(out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_uma.avg.pct_of_peak_sustained_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size", "launch__shared_mem_per_block_dynamic",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "lts__t_bytes.sum",
        "smsp__average_warp_latency_issue_stalled_long_scoreboard", "sm__cycles_elapsed.avg"]


def full(path: str, out: str, alg_bytes: float | None = None, alg_flops: float | None = None) -> None:
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw[raw.index('"ID"'):])))
    h, units = rows[0], rows[1]
    lines = [f"# ncu --set full: `{path.split('/')[-1]}`", ""]
    for r in rows[2:]:
        d = dict(zip(h, r))
        u = dict(zip(h, units))
        lines.append(f"## `{short(d.get('Kernel Name', '?'))}` grid {d.get('launch__grid_size')} x block "
                     f"{d.get('launch__block_size')}")
        lines.append("")
        lines.append("| metric | value | unit |")
        lines.append("|---|---:|---|")
        for k in KEYS:
            if k in d and d[k] != "":
                lines.append(f"| `{k}` | {d[k]} | {u.get(k, '')} |")
        try:
            dur_ns = float(d["gpu__time_duration.sum"].replace(",", "")) * (1e3 if u["gpu__time_duration.sum"] == "us"
                                                                            else 1.0)
            scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
            rd = float(d["dram__bytes_read.sum"].replace(",", "")) * scale.get(u["dram__bytes_read.sum"], 1)
            wr = float(d["dram__bytes_write.sum"].replace(",", "")) * scale.get(u["dram__bytes_write.sum"], 1)
            lines.append("")
            lines.append(f"DRAM traffic per launch: {(rd + wr) / 1e6:.2f} MB (read {rd / 1e6:.2f}, write {wr / 1e6:.2f});"
                         f" {(rd + wr) / dur_ns:.1f} GB/s over {dur_ns / 1e3:.1f} µs.")
            if alg_bytes:
                lines.append(f"Algorithmic bytes {alg_bytes / 1e6:.2f} MB -> traffic/algorithmic = "
                             f"{(rd + wr) / alg_bytes:.2f}; achieved {alg_bytes / dur_ns:.1f} GB/s.")
            if alg_flops:
                lines.append(f"Algorithmic FLOPs {alg_flops / 1e9:.2f} G -> {alg_flops / dur_ns / 1e3:.1f} TFLOP/s.")
        except (KeyError, ValueError):
            pass
        lines.append("")
    open(out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        launches(sys.argv[2], sys.argv[3])
    else:
        full(sys.argv[2], sys.argv[3], *(float(x) for x in sys.argv[4:6]))
