#!/usr/bin/env python
"""Summarises EMBER_TC_CTATIMES=<file> (per-CTA %globaltimer start/end of one warmed-up rows + dN
launch, [2 launches][sm_count][start, end] ns) as the table rows of profiles/r02_rows_cta_spans.md."""
import sys

import numpy as np


def main(path, sm=148):
    raw = np.fromfile(path, dtype=np.uint64).astype(np.int64)
    rows, dn = raw[:2 * sm].reshape(-1, 2), raw[2 * sm:4 * sm].reshape(-1, 2)
    rows, dn = rows[rows[:, 0] > 0], dn[dn[:, 0] > 0]
    t0 = rows[:, 0].min()
    for name, x in (("rows `k_tc<0>`", rows), ("dN `k_tc<1>`", dn)):
        s, e = (x[:, 0] - t0) / 1e3, (x[:, 1] - t0) / 1e3
        print(f"| {name} | {len(x)} | {int((s > s.min() + 1).sum())} | {s.max():.1f} | {e.min():.1f} | "
              f"{np.median(e):.1f} | {e.max():.1f} |")
    e = (rows[:, 1] - t0) / 1e3
    h, b = np.histogram(e, bins=10)
    print("| " + " | ".join(f"{b[i]:.0f}-{b[i + 1]:.0f}" for i in range(10)) + " |")
    print("| " + " | ".join(str(v) for v in h) + " |")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 148)
