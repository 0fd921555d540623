#!/usr/bin/env python
"""Run-length statistics of one bench batch's gradient keys (relations, source / destination nodes):
how many keys repeat, how many take the long-segment path (> EMBER_LONG_SEG rows) and the largest
runs. Negatives are left out (they add 2,000 mostly-distinct rows)."""
import sys

import torch

sys.path.insert(0, ".")
import bench  # noqa: E402

cfg = bench.CONFIGS["fb86m"]
W = bench.Workload(cfg, 0, "tc")
n = len(W.batches) // 3
lo, hi, begin, nb, i, j, step, k = W.batches[n]
e = W.edges[lo + begin: lo + begin + nb].long()
for name, col in (("src", 0), ("rel", 1), ("dst", 2)):
    keys = e[:, col]
    if name != "rel":  # node keys of both sides share a key space
        pass
    u, c = torch.unique(keys, return_counts=True)
    c = c.sort(descending=True).values
    rep = c[c > 1]
    lng = c[c > 16]
    print(f"{name}: rows {nb} unique {len(u)} repeated-keys {len(rep)} rows-in-repeated {int(rep.sum())} "
          f"long(>16) {len(lng)} rows-in-long {int(lng.sum())} chunks {int(((lng + 31) // 32).sum())} top {c[:8].tolist()}")
nodes = torch.cat([e[:, 0], e[:, 2]])
u, c = torch.unique(nodes, return_counts=True)
c = c.sort(descending=True).values
print(f"nodes(both sides): unique {len(u)} repeated {(c > 1).sum().item()} long {(c > 16).sum().item()} top {c[:8].tolist()}")
