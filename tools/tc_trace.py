#!/usr/bin/env python
"""Reads a k_tc CTA-0 timeline (EMBER_TC_TRACE=<prefix> -> <prefix>.rows.bin / .negs.bin) and
prints per-tile latencies of the MMA <-> epilogue handshake (cycles, SM clock)."""
import collections
import sys

import numpy as np

NAMES = {1: "P.res_load", 2: "P.ring_slot", 10: "M.R_ready", 11: "M.ring_full", 12: "M.S_issued", 13: "M.P_full",
         14: "M.PN_issued", 15: "M.acc_empty", 16: "M.ring_wait", 17: "M.P_wait", 20: "E0.S_full", 21: "E1.S_full", 22: "E0.P_done", 23: "E1.P_done",
         24: "E0.stage_start", 25: "E0.stage_end", 26: "E0.acc_full", 27: "E1.acc_full", 28: "E0.tail_end",
         29: "E1.tail_end", 30: "E1.acc_ld0", 31: "E1.acc_ld1", 32: "E1.z_ready"}


def main(path, show=120):
    raw = np.fromfile(path, dtype=np.uint64).reshape(-1, 2)
    raw = raw[raw[:, 0] != 0]  # unused slots of the per-role regions
    t = raw[:, 0].astype(np.int64)
    ev = (raw[:, 1] >> 32).astype(np.int64)
    arg = (raw[:, 1] & 0xFFFFFFFF).astype(np.int64)
    o = np.argsort(t, kind="stable")
    t, ev, arg = t[o] - t[o][0], ev[o], arg[o]
    first = collections.defaultdict(dict)
    for ti, e, a in zip(t, ev, arg):
        first[e].setdefault(a, ti)
    print(f"{len(t)} events over {t[-1]} cycles")
    for ti, e, a in list(zip(t, ev, arg))[:show]:
        print(f"{ti:9d}  {NAMES.get(e, e):16s} {a}")

    def lat(e1, e2, label):
        d = [first[e2][a] - first[e1][a] for a in first[e1] if a in first[e2]]
        if d:
            print(f"{label:44s} n={len(d):4d} median {np.median(d):8.0f}  mean {np.mean(d):8.0f}")

    s_full = {**first[20], **first[21]}
    p_done = {**first[22], **first[23]}
    first[100] = s_full
    first[101] = p_done
    lat(12, 100, "S issued -> epilogue sees S_full")
    lat(100, 101, "epilogue: S_full -> P written (T_E)")
    lat(101, 13, "P written -> MMA sees P_full")
    lat(13, 14, "MMA: P_full -> PN issued")
    lat(11, 12, "MMA: ring_full -> S issued")
    iss = np.array(sorted(first[12].values()))
    if len(iss) > 2:
        print(f"{'S issue period':44s} median {np.median(np.diff(iss)):8.0f}  mean {np.mean(np.diff(iss)):8.0f}")
    lat(27, 32, "tail: acc_full -> z ready")
    lat(32, 30, "tail: z ready -> acc batch 0 loaded")
    lat(30, 31, "tail: batch 0 stores + batch 1 loaded")
    lat(31, 29, "tail: batch 1 stores -> tail end")
    rf = first[11]
    prev = {q: first[12].get(q - 1) for q in rf}
    d = [rf[q] - prev[q] for q in rf if prev[q] is not None]
    if d:
        print(f"{'MMA wait for ring (prev S issued -> ring_full)':44s} median {np.median(d):8.0f} mean {np.mean(d):8.0f}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 120)
