#!/usr/bin/env python
"""Per-kernel counts of the SASS instructions that prove the tensor-core / TMA / async-copy paths
(cuobjdump -sass of the built library): UTCHMMA/UTCQMMA (tcgen05.mma), UTCCP (tcgen05.cp), LDTM/STTM
(tcgen05.ld/st), UTMALDG (TMA tensor loads), UBLKCP (bulk copies), LDGSTS (cp.async), plus the size.
usage: python tools/sass_summary.py [lib.so] > profiles/<round>_sass_summary.md"""
import collections
import re
import subprocess
import sys

lib = sys.argv[1] if len(sys.argv) > 1 else "paper_2101_08358_b200/libember_b200.so"
out = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True, check=True).stdout
OPS = ["UTCHMMA", "UTCQMMA", "UTCCP", "LDTM", "STTM", "UTMALDG", "UBLKCP", "LDGSTS", "SYNCS", "ELECT"]
kern = None
counts = collections.OrderedDict()
for line in out.splitlines():
    m = re.match(r"\s*Function : (\S+)", line)
    if m:
        kern = m.group(1)
        counts[kern] = collections.Counter()
        continue
    if kern is None:
        continue
    m = re.search(r"/\*[0-9a-f]{4,}\*/\s+(@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)", line)
    if m:
        op = m.group(2)
        counts[kern]["_insts"] += 1
        for o in OPS:
            if op.startswith(o):
                counts[kern][o] += 1


def demangle(names):
    r = subprocess.run(["c++filt"], input="\n".join(names), capture_output=True, text=True)
    return r.stdout.splitlines() if r.returncode == 0 else names


def clean(p):
    p = p.replace("(anonymous namespace)::", "").replace("ember::", "")
    p = re.sub(r"^void ", "", p)
    p = re.sub(r"cub::CUB_\w+::", "cub::", p)
    return re.sub(r"\(.*", "", re.sub(r"<(?:[^<>]|<[^<>]*>)*>", lambda m: m.group(0) if len(m.group(0)) < 12 else "<...>", p))


names = list(counts)
pretty = demangle(names)
print(f"# SASS summary of `{lib}` (cuobjdump -sass, sm_100a)\n")
print("| kernel | insts | " + " | ".join(OPS) + " |")
print("|---|---:|" + "---:|" * len(OPS))
for n, p in zip(names, pretty):
    c = counts[n]
    if not any(c[o] for o in OPS):
        continue
    p = clean(p)
    print(f"| `{p}` | {c['_insts']} | " + " | ".join(str(c[o]) for o in OPS) + " |")
others = [clean(p) for n, p in zip(names, pretty) if not any(counts[n][o] for o in OPS)]
print(f"\nKernels without any of these instructions ({len(others)}): " + ", ".join(f"`{o}`" for o in others[:80]))
