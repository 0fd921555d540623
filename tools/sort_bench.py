"""Warm timing of the step's hand-written (key, slot) sort (ember_debug_sort_slots, runs included) on the
FB86m bench's slot shape, beside torch.sort(stable) of the same keys (CUB onesweep: the library sort
it replaced, without the run-length pass). CUDA events on the context stream around 200 back-to-back calls."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2101_08358_b200 as eb  # noqa: E402

tr = eb.Trainer(eb.Hyper(kind="complex", dim=16, batch_size=50000, num_negatives=1000, engine="tc"), 3000, 20, 1,
                device=0)
tr.init_embeddings(11)
rng = np.random.default_rng(1)
nb, n_neg, node_range = 50000, 2000, 10_757_000
z = rng.zipf(1.2, size=2 * nb + n_neg).astype(np.uint64) - 1
nodes = ((z * 2654435761) % node_range).astype(np.uint32)
zr = rng.zipf(1.5, size=nb).astype(np.uint64) - 1
rels = (node_range + (zr * 2654435761) % 14824).astype(np.uint32)
keys = np.concatenate([nodes, rels])
dk = torch.from_numpy(keys.view(np.int32)).cuda()
from paper_2101_08358_b200 import _lib  # noqa: E402

lib = eb.lib()
n = len(keys)
nruns = torch.zeros(1, dtype=torch.int32, device="cuda")
st = torch.cuda.Stream(device=0)


def one():
    assert lib.ember_debug_sort_slots(tr.ctx, dk.data_ptr(), n, 24, None, None, None, None, None, None,
                                      nruns.data_ptr()) == 0


for _ in range(20):
    one()
tr.synchronize()
torch.cuda.synchronize()
import time  # noqa: E402

reps = 200
cs = torch.cuda.ExternalStream(lib.ember_ctx_stream(tr.ctx))
a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
t0 = time.perf_counter()
a0.record(cs)
for _ in range(reps):
    one()
a1.record(cs)
tr.synchronize()
host = (time.perf_counter() - t0) / reps * 1e6
ours = a0.elapsed_time(a1) / reps * 1e3
kt = torch.from_numpy(keys.astype(np.int64)).cuda()
for _ in range(20):
    torch.sort(kt, stable=True)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
k32 = dk.clone()
e0.record()
for _ in range(reps):
    torch.sort(k32, stable=True)
e1.record()
torch.cuda.synchronize()
print(f"slot sort (hand-written, incl. runs + key copy): device {ours:.1f} us/call (host {host:.1f}); "
      f"torch.sort stable int32 (CUB): {e0.elapsed_time(e1) / reps * 1e3:.1f} us/call; n={n} nruns={int(nruns.item())}")
