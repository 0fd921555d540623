#!/usr/bin/env python
"""bench.py — train edges/sec of the B200-native Gaius/Marius minibatch training step.

Metric (BASELINE.json): train edges/sec at 1/2/4/8 B200, Freebase86m-shaped ComplEx d=100,
16 partitions, BETA (elimination) ordering; b=5e4, n_t=1e3, alpha=0.5, lr=0.1.

A "step" is one training batch (sample -> gather -> scores/LSE/gradients -> Adagrad) taken in
BETA bucket order from a synthetic graph of the named shape, parameters resident in HBM.
  value : edges/s with inputs already in HBM, CUDA events on the step stream, max over ranks.
  e2e   : the same steps through the host-buffer C-ABI call (ember_train_batch_host): every step
          copies its positives from pinned host memory and reads its loss back.
  --impl reference: the reference's CPU training step (its SPEC restated in oracle/; the reference
          ships no runnable trainer) on the host cores: same graph, plan and full batches as the GPU
          arm's timed window, sampling + dedupe + gather + loss_and_grad + Adagrad per step; never
          loads the product library.
Usage: python bench.py [--gpus N] [--steps K] [--warmup W] [--config fb86m] [--engine tc|simt]
"""
from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    # name: |V|, |R|, |E| (all splits), model, d, b, n_t, alpha, partitions, train/valid fractions
    "fb86m": dict(V=86_054_151, R=14_824, E=338_586_276, kind="complex", dim=100, b=50_000, nt=1000, alpha=0.5,
                  p=16, train=0.9, valid=0.05,
                  desc="Freebase86m-shaped KG, ComplEx d=100, 16 partitions, BETA ordering"),
    "livejournal": dict(V=4_847_571, R=1, E=68_993_773, kind="dot", dim=100, b=50_000, nt=1000, alpha=0.5, p=1,
                        train=0.9, valid=0.05, desc="LiveJournal-shaped social graph, Dot d=100, in-memory"),
    "fb15k237": dict(V=14_541, R=237, E=340_144, kind="distmult", dim=100, b=10_000, nt=1000, alpha=0.5, p=1,
                     train=0.8, valid=0.1, desc="FB15k-237-shaped KG, DistMult d=100, in-memory"),
    "twitter": dict(V=41_652_230, R=1, E=1_468_365_182, kind="dot", dim=100, b=50_000, nt=1000, alpha=0.5, p=16,
                    train=0.9, valid=0.05, desc="Twitter-shaped graph, Dot d=100, 16 partitions"),
    "fb86m_d800": dict(V=86_054_151, R=14_824, E=338_586_276, kind="complex", dim=800, b=50_000, nt=1000, alpha=0.5,
                       p=16, train=0.9, valid=0.05, desc="Freebase86m-shaped KG, ComplEx d=800, 16 partitions"),
    # C5's step (d = 800, b, n_t, |R| as C3) on 1/8 of the nodes and edges, so the 68.8 GB of tables
    # fit one GPU; run with --engine simt (the tensor-core TMEM layout stops at d = 128)
    "fb86m_d800_step": dict(V=10_756_769, R=14_824, E=42_323_284, kind="complex", dim=800, b=50_000, nt=1000,
                            alpha=0.5, p=16, train=0.9, valid=0.05,
                            desc="C5 step shape (ComplEx d=800, b=5e4, n_t=1e3) on 1/8 of Freebase86m's nodes/edges"),
}
METRIC = "train edges/sec (Freebase86m-shape ComplEx d=100, 16 partitions, BETA ordering)"
GRAPH_SEED, INIT_SEED, NEG_SEED, ORDER_SEED = 210108358, 11, 1, 0


def peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0, "_fallback": True}


def executed_tc_flops(cfg, nb):
    """Tensor-pipe FLOPs the bf16x3 engine executes per step (csrc/tc_score.cu): every 96-wide
    streamed tile of either kernel runs S (128 x 96 x KP) and P.T (128 x KP x 96), 3 MMAs each
    (hi.hi + hi.lo + lo.hi); rows kernel: 2 sides x ceil(nb/128) items x ceil(nt/96) tiles; negs
    kernel (recomputes S): 2 sides x ceil(nt/128) x ceil(nb/96) tiles; KP = d rounded up to 16."""
    d, nt = cfg["dim"], cfg["nt"]
    kp = (d + 15) // 16 * 16
    c = lambda a, b: -(-a // b)  # noqa: E731
    tiles = 2 * c(nb, 128) * c(nt, 96) + 2 * c(nt, 128) * c(nb, 96)
    return tiles * 2 * (2 * 128 * 96 * kp) * 3


def algorithmic(cfg):
    """Per-edge algorithmic work: FLOPs = 3 contractions x 2 sides x 2*n_t*d;
    HBM bytes = 12 + 32d + 32d*n_t/b (nominal: unique rows touched read+write theta and acc)."""
    d, nt, b = cfg["dim"], cfg["nt"], cfg["b"]
    return 12.0 * nt * d, 12.0 + 32.0 * d + 32.0 * d * nt / b


# ------------------------------------------------------------------------------ clocks

class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.proc = None
        self.lines: list[str] = []

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.th = threading.Thread(target=self._read, daemon=True)
            self.th.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self) -> dict:
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx.append(float(f[2]))
            except ValueError:
                continue
            for n, v in zip(names, f[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ------------------------------------------------------------------------------ workload

class Workload:
    """Synthetic graph of the config's shape, bucketed, with tables initialised on this GPU."""

    def __init__(self, cfg, device, engine, rank=0, world=1):
        import torch

        import paper_2101_08358_b200 as eb
        self.eb, self.torch, self.cfg = eb, torch, cfg
        self.device = device
        p = cfg["p"]
        n_total = cfg["E"]
        edges, split = eb.generate_graph(cfg["V"], cfg["R"], n_total, GRAPH_SEED, cfg["train"], cfg["valid"],
                                         device=device)
        train = edges[split == 0]
        del edges, split
        self.edges, self.offsets = eb.bucket_edges(train, cfg["V"], p, device=device)
        del train
        torch.cuda.empty_cache()
        self.n_train = int(self.offsets[-1])
        h = eb.Hyper(kind=cfg["kind"], dim=cfg["dim"], batch_size=cfg["b"], num_negatives=cfg["nt"],
                     alpha=cfg["alpha"], neg_seed=NEG_SEED, engine=engine)
        self.tr = eb.Trainer(h, cfg["V"], cfg["R"], p, device=device)
        self.tr.init_embeddings(INIT_SEED)
        self.plan = eb.make_plan("elimination", p, p, ORDER_SEED)  # all partitions resident: c = p
        self.batches = batch_list(self.plan["seq"], self.offsets, p, cfg["b"])
        self.base = self.edges.data_ptr()
        torch.cuda.synchronize()

    def batch_args(self, n):
        lo, hi, begin, nb, i, j, step, k = self.batches[n % len(self.batches)]
        return self.base + 12 * lo, hi - lo, begin, nb, i, j, step, k

    def run_steps(self, start, count, epoch=0):
        eb = self.eb
        L = eb.lib()
        edges = 0
        for n in range(start, start + count):
            ptr, bn, begin, nb, i, j, step, k = self.batch_args(n)
            eb.check(L.ember_train_batch(self.tr.ctx, ptr, bn, begin, nb, i, j, epoch, step, k, None))
            edges += nb
        return edges


def dist_partitions(cfg, world):
    """Partitions of the multi-GPU path: the overlapped (coset) schedule needs p a power of two with
    world | p/4, so p = max(config p, 4 * world) (FB86m at 8 GPUs: 32 partitions of 2.15 GB)."""
    p = cfg["p"]
    while p < 4 * world or p & (p - 1):
        p += 1
    return p


def bench_distributed(args, rank, world, local_rank):
    """N > 1 (or --distributed at N = 1): one process per GPU through the library's multi-GPU driver
    (ember_dist_*: C++ round loop, csrc/host/dist_driver.cpp + csrc/dist.cu). Each rank holds
    p/N partitions in driver-owned HBM slots, trains its buckets of the round, sums relation
    gradients with an NCCL all-reduce on the step stream every (lockstep) step, and hands partitions
    to their next holder with NCCL send/recv on a copy stream (second communicator) issued right
    after the departing pair's buckets, under the staying pair's steps (overlapped coset schedule).
    Timed: K lockstep steps after W warm-up steps from the epoch's start (self-buckets, handoffs
    and idle steps included); value = real edges of all ranks / max-over-ranks device time.
    torch.distributed only shares the two NCCL unique ids and the final timings."""
    import torch
    import torch.distributed as dist

    import paper_2101_08358_b200 as eb
    from paper_2101_08358_b200 import distributed as ed
    cfg = dict(CONFIGS[args.config])
    cfg["p"] = dist_partitions(cfg, world)
    torch.cuda.set_device(local_rank)
    edges, split = eb.generate_graph(cfg["V"], cfg["R"], cfg["E"], GRAPH_SEED, cfg["train"], cfg["valid"],
                                     device=local_rank)
    train = edges[split == 0]
    del edges, split
    bucketed, offsets = eb.bucket_edges(train, cfg["V"], cfg["p"], device=local_rank)
    del train
    torch.cuda.empty_cache()
    h = eb.Hyper(kind=cfg["kind"], dim=cfg["dim"], batch_size=cfg["b"], num_negatives=cfg["nt"], alpha=cfg["alpha"],
                 neg_seed=NEG_SEED, engine=args.engine)
    tr = eb.Trainer(h, cfg["V"], cfg["R"], cfg["p"], device=local_rank, allocate=False)
    ids = None
    if world > 1:
        idt = torch.zeros(256, dtype=torch.uint8, device="cuda")
        if rank == 0:
            idt.copy_(torch.frombuffer(bytearray(ed.nccl_unique_id() + ed.nccl_unique_id()), dtype=torch.uint8))
        dist.broadcast(idt, 0)
        raw = bytes(idt.cpu().numpy().tobytes())
        ids = (raw[:128], raw[128:])
    D = ed.NativeDistributed(tr, bucketed, offsets, rank, world, overlap=True, ids=ids)
    D.init_embeddings(INIT_SEED)
    stream = tr.torch_stream()
    total = D.total_steps()
    K = min(args.steps, total - args.warmup)
    D.run_steps(0, args.warmup, 0)
    D.synchronize()
    p0 = tr.profile_read()  # launch counters only: phase events stay off in the timed region
    launches0 = p0["launches"]
    dist.barrier()
    torch.cuda.synchronize()
    clocks = ClockSampler(local_rank)
    clocks.start()
    time.sleep(0.3)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    rep = D.run_steps(args.warmup, K, 0)
    e1.record(stream)
    D.synchronize()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    clk = clocks.stop()
    p1 = tr.profile_read()
    launches = p1["launches"] - launches0
    n_edges = int(rep.edges)
    # e2e: the next K steps with their positives copied in from pinned host memory inside the timed
    # region (this rank's batches of those steps, one async copy each, in step order), and the last
    # step's loss read back
    start2 = args.warmup + K
    K2 = min(K, total - start2)
    host = bucketed.cpu().pin_memory()
    spans, step = [], 0
    for r in range(D.plan.rounds):
        mine = ed.round_batches(D.plan, offsets, cfg["b"], r, rank)
        for s in range(D.steps_per_round[r]):
            if start2 <= step < start2 + K2 and s < len(mine):
                _, _, _, _, lo, _, begin, nb = mine[s]
                spans.append((lo + begin, nb))
            step += 1
    dist.barrier()
    torch.cuda.synchronize()
    h0 = time.perf_counter()
    with torch.cuda.stream(stream):
        for a, n in spans:
            bucketed[a:a + n].copy_(host[a:a + n], non_blocking=True)
    rep2 = D.run_steps(start2, K2, 0) if K2 > 0 else None
    loss = D.loss()
    e2e_ms = (time.perf_counter() - h0) * 1e3
    e2e_edges = int(rep2.edges) if rep2 else 0
    h2d = sum(n for _, n in spans) * 12
    assert np.isfinite(loss)
    vals = torch.tensor([ms, e2e_ms], dtype=torch.float64, device="cuda")
    dist.all_reduce(vals, op=dist.ReduceOp.MAX)
    tot = torch.tensor([float(n_edges), float(e2e_edges), float(rep.handoff_bytes), float(h2d),
                        float(rep.early_handoffs), float(rep.handoffs)], dtype=torch.float64, device="cuda")
    dist.all_reduce(tot, op=dist.ReduceOp.SUM)
    ms, e2e_ms = float(vals[0]), float(vals[1])
    n_edges, e2e_edges = float(tot[0]), float(tot[1])
    D.close()
    if rank != 0:
        return None
    flops_e, bytes_e = algorithmic(cfg)
    return {
        "metric": METRIC if args.config == "fb86m" else f"train edges/sec ({cfg['desc']})",
        "value": round(n_edges / (ms / 1e3), 1), "unit": "edges/s", "n_gpus": world, "steps": K,
        "warmup": args.warmup, "ms_per_step": round(ms / K, 4), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32 (bf16x3 split on tensor cores)" if args.engine == "tc" else "f32",
        "data": "synthetic (planted-community power-law graph of the named shape; random-init Adagrad state)",
        "config": {"workload": cfg["desc"], "nodes": cfg["V"], "relations": cfg["R"], "edges_total": cfg["E"],
                   "train_edges": int(offsets[-1]), "model": cfg["kind"], "dim": cfg["dim"], "batch": cfg["b"],
                   "negatives_per_side": cfg["nt"], "partitions": cfg["p"],
                   "ordering": "overlapped coset rounds (ember_make_rounds_overlap)", "engine": args.engine,
                   "parallelism": f"partition-sharded x{world} (library driver: NCCL relation all-reduce on the "
                                  f"step stream, NCCL P2P handoff on a copy stream)",
                   "l2": "inputs larger than L2 (node tables, random rows per batch)",
                   "steps_per_round": D.steps_per_round[1] if len(D.steps_per_round) > 1 else D.steps_per_round[0],
                   "handoff_bytes_timed": int(float(tot[2])), "handoffs_timed": int(float(tot[5])),
                   "handoffs_before_round_end": int(float(tot[4]))},
        "e2e": {"value": round(e2e_edges / (e2e_ms / 1e3), 1) if e2e_ms > 0 else None, "unit": "edges/s",
                "h2d_bytes_per_step": int(float(tot[3]) / max(1, K2) / world), "d2h_bytes_per_step": 4,
                "timing": "host clock: pinned-host copies of the window's positives, the driver call, the loss read-back"},
        "gpu_launches": int(launches),
        "roofline": None,
        "clocks": clk,
    }


def bench_buffered(args, local_rank):
    """--capacity c < p: the device partition buffer (csrc/buffer.cu): c HBM slots (+2 staging) over
    the pinned host backing store, BETA plan for (p, c), prefetch + async writeback on copy streams.
    One warm-up epoch, then one timed epoch (CUDA events on the step stream, stalls included)."""
    import torch

    import paper_2101_08358_b200 as eb
    cfg = CONFIGS[args.config]
    p, c = cfg["p"], args.capacity
    torch.cuda.set_device(local_rank)
    edges, split = eb.generate_graph(cfg["V"], cfg["R"], cfg["E"], GRAPH_SEED, cfg["train"], cfg["valid"],
                                     device=local_rank)
    train = edges[split == 0]
    del edges, split
    bucketed, offsets = eb.bucket_edges(train, cfg["V"], p, device=local_rank)
    del train
    torch.cuda.empty_cache()
    h = eb.Hyper(kind=cfg["kind"], dim=cfg["dim"], batch_size=cfg["b"], num_negatives=cfg["nt"], alpha=cfg["alpha"],
                 neg_seed=NEG_SEED, engine=args.engine)
    tr = eb.Trainer(h, cfg["V"], cfg["R"], p, device=local_rank, allocate=False)
    plan = eb.make_plan("elimination", p, c, ORDER_SEED)
    t0 = time.perf_counter()
    buf = eb.PartitionBuffer(tr, c, plan["seq"])
    buf.init_backing(INIT_SEED)
    setup_s = time.perf_counter() - t0
    stream = tr.torch_stream()
    buf.train_epoch(bucketed, offsets, 0)
    buf.flush()
    torch.cuda.synchronize()
    st0 = buf.stats()
    clocks = ClockSampler(local_rank)
    clocks.start()
    time.sleep(0.3)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    out = buf.train_epoch(bucketed, offsets, 1)
    buf.flush()  # the step stream waits for the epoch-end writebacks: they are inside the timed region
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    clk = clocks.stop()
    st = buf.stats()
    n = out["edges"]
    gb = (st["bytes_read"] - st0["bytes_read"] + st["bytes_written"] - st0["bytes_written"]) / 1e9
    return {"metric": f"train edges/sec through the partition buffer ({cfg['desc']}, c={c})", "value": round(n / (ms / 1e3), 1),
            "unit": "edges/s", "n_gpus": 1, "steps": int(out["batches"]), "warmup": "1 epoch",
            "ms_per_step": round(ms / max(1, out["batches"]), 4), "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f32 (bf16x3 split on tensor cores)" if args.engine == "tc" else "f32",
            "data": "synthetic", "config": {"workload": cfg["desc"], "partitions": p, "buffer_capacity": c,
                                            "ordering": "elimination (BETA)", "engine": args.engine,
                                            "backing_store": "pinned host memory", "timed": "one full epoch"},
            "buffer": {"swaps_per_epoch": st["swaps_per_epoch"], "plan_swap_count": plan["swap_count"],
                       "reads_epoch": st["reads"] - st0["reads"], "writes_epoch": st["writes"] - st0["writes"],
                       "pcie_gb_epoch": round(gb, 2), "stall_ms_epoch": round(st["stall_ms"] - st0["stall_ms"], 3),
                       "stalls_epoch": st["stalls"] - st0["stalls"], "slots": st["slots"],
                       "slot_gb": round(st["slot_bytes"] / 1e9, 2), "setup_s": round(setup_s, 1)},
            "epoch_s": round(ms / 1e3, 3), "loss": out["loss"], "clocks": clk}


def bench_ours(args, rank, world, local_rank):
    import torch
    import torch.distributed as dist
    cfg = CONFIGS[args.config]
    torch.cuda.set_device(local_rank)
    W = Workload(cfg, local_rank, args.engine, rank, world)
    tr, eb = W.tr, W.eb
    stream = tr.torch_stream()
    start_at = len(W.batches) // 3  # steady state: middle of the epoch's bucket sequence

    W.run_steps(start_at, args.warmup)
    torch.cuda.synchronize()
    p0 = tr.profile_read()  # (phase events stay off in the timed region)
    launches0, lib0 = p0["launches"], p0["lib_calls"]
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clocks = ClockSampler(local_rank)
    clocks.start()
    time.sleep(0.3)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.profiler.start()  # ncu --profile-from-start off captures exactly the timed steps
    e0.record(stream)
    edges = W.run_steps(start_at + args.warmup, args.steps)
    e1.record(stream)
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()
    ms = e0.elapsed_time(e1)
    clk = clocks.stop()
    p1 = tr.profile_read()
    launches, lib_calls = p1["launches"] - launches0, p1["lib_calls"] - lib0

    # e2e: same steps through the host-buffer call, positives copied from pinned host memory
    host_batches = []
    for n in range(start_at + args.warmup, start_at + args.warmup + args.steps):
        ptr, bn, begin, nb, i, j, step, k = W.batch_args(n)
        lo = W.batches[n % len(W.batches)][0]
        t = W.edges[lo + begin: lo + begin + nb].cpu().pin_memory()
        host_batches.append((t, ptr, bn, nb, i, j, step, k))
    loss_host = torch.zeros(len(host_batches), dtype=torch.float32).pin_memory()
    L = eb.lib()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    # timed on the host clock from the first call to the return of ember_ctx_synchronize (every
    # stream of the context, the loss read-backs included); the device-event span is kept beside it
    x0, x1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    h0 = time.perf_counter()
    x0.record(stream)
    e2e_edges = h2d = 0
    for s, (t, ptr, bn, nb, i, j, step, k) in enumerate(host_batches):
        eb.check(L.ember_train_batch_host(tr.ctx, ptr, bn, t.data_ptr(), nb, i, j, 1, step, k,
                                          loss_host.data_ptr() + 4 * s))
        e2e_edges += nb
        h2d += nb * 12
    x1.record(stream)
    eb.check(L.ember_ctx_synchronize(tr.ctx))
    e2e_ms = (time.perf_counter() - h0) * 1e3
    torch.cuda.synchronize()
    e2e_device_ms = x0.elapsed_time(x1)
    assert np.isfinite(loss_host.numpy()).all()

    # phase breakdown: the next K steps again with CUDA events at the phase boundaries (the events
    # serialise the programmatic launches, so this pass is not the timed one)
    tr.profile(True)
    tr.profile_read()
    W.run_steps(start_at + args.warmup + 2 * args.steps, args.steps)
    prof = tr.profile_read()
    tr.profile(False)

    # max over ranks
    vals = torch.tensor([ms, e2e_ms, float(edges), float(e2e_edges)], dtype=torch.float64, device="cuda")
    if world > 1:
        t_max = vals[:2].clone()
        dist.all_reduce(t_max, op=dist.ReduceOp.MAX)
        tot = vals[2:].clone()
        dist.all_reduce(tot, op=dist.ReduceOp.SUM)
        ms, e2e_ms = float(t_max[0]), float(t_max[1])
        edges, e2e_edges = float(tot[0]), float(tot[1])
    if rank != 0:
        return None

    flops_e, bytes_e = algorithmic(cfg)
    pk = peaks()
    contract_ms = prof["ms"]["contraction"] / max(1, args.steps)
    step_edges = edges / max(1, args.steps) / world
    achieved = flops_e * step_edges / (contract_ms / 1e3) / 1e12 if contract_ms > 0 else None
    exe = (executed_tc_flops(cfg, cfg["b"]) / (contract_ms / 1e3) / 1e12
           if contract_ms > 0 and args.engine == "tc" else None)
    # the contraction runs inside a 0.35 ms step at the maximum SM clock (clocks below): the burst
    # peak is its denominator; the power-capped sustained figure is reported beside it
    peak = pk.get("bf16_tflops")
    peak_s = pk.get("bf16_tflops_sustained", peak)
    traffic, ncu = None, {}
    prof_file = os.path.join(ROOT, "profiles", f"ncu_summary_{args.engine}.json")
    if os.path.exists(prof_file):
        try:
            ncu = json.load(open(prof_file))
            traffic = ncu.get("dram_bytes_per_launch")
        except Exception:
            ncu = {}
    value = edges / (ms / 1e3)
    # memory-bound phases: this run's phase times against the DRAM bytes ncu measured for the same
    # kernels (profiles/ncu_summary_<engine>.json, one cold-cache launch each)
    hbm_phases = {}
    for ph, mb in (ncu.get("phase_dram_mb") or {}).items():
        t_ms = prof["ms"].get(ph, 0.0) / max(1, args.steps)
        if t_ms > 0:
            gbs = mb * 1e6 / (t_ms / 1e3) / 1e9
            hbm_phases[ph] = {"ms": round(t_ms, 4), "dram_mb": mb, "gbs": round(gbs, 1),
                              "frac": round(gbs / pk["hbm_gbs"], 4), "kernels": ncu.get("phase_kernels", {}).get(ph)}
    out = {
        "metric": METRIC if args.config == "fb86m" else f"train edges/sec ({cfg['desc']})",
        "value": round(value, 1),
        "unit": "edges/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(ms / args.steps, 4),
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "f32 (bf16x3 split on tensor cores)" if args.engine == "tc" else "f32",
        "data": "synthetic (planted-community power-law graph of the named shape; random-init Adagrad state)",
        "config": {"workload": cfg["desc"], "nodes": cfg["V"], "relations": cfg["R"], "edges_total": cfg["E"],
                   "train_edges": W.n_train, "model": cfg["kind"], "dim": cfg["dim"], "batch": cfg["b"],
                   "negatives_per_side": cfg["nt"], "alpha": cfg["alpha"], "partitions": cfg["p"],
                   "buffer_capacity": cfg["p"], "ordering": "elimination (BETA)", "engine": args.engine,
                   "l2": "inputs larger than L2 (node tables %.1f GB, random rows per batch)"
                         % (cfg["V"] * cfg["dim"] * 8 / 1e9),
                   "parallelism": f"partition-sharded x{world}" if world > 1 else "1 GPU"},
        "e2e": {"value": round(e2e_edges / (e2e_ms / 1e3), 1), "unit": "edges/s",
                "h2d_bytes_per_step": int(h2d / max(1, len(host_batches))), "d2h_bytes_per_step": 4,
                "timing": "host clock: first ember_train_batch_host call to the return of ember_ctx_synchronize",
                "device_span_ms_per_step": round(e2e_device_ms / max(1, len(host_batches)), 4)},
        "gpu_launches": int(launches),
        "library_calls": int(lib_calls),
        "phase_ms_per_step": {k: round(v / args.steps, 4) for k, v in prof["ms"].items()},
        "roofline": {"bound": "tensor", "kernel": "contraction (scores + LSE + dA + dN)",
                     "achieved": round(achieved, 2) if achieved else None, "peak": peak, "unit": "TFLOP/s",
                     "frac": round(achieved / peak, 4) if achieved else None, "traffic": traffic,
                     "frac_sustained": round(achieved / peak_s, 4) if achieved else None,
                     "flops_per_edge": flops_e, "peak_source": "MEASURED_PEAKS.json bf16_tflops (burst: the step "
                     "runs at the maximum SM clock); frac_sustained uses bf16_tflops_sustained"
                     + (" (fallback)" if pk.get("_fallback") else ""),
                     "traffic_source": ncu.get("source"),
                     # the fp32-accurate bf16x3 scheme executes ~4.7x the algorithmic FLOPs (3 MMAs per
                     # product, S recomputed by the dN kernel, K and N padding): tensor-pipe utilisation
                     "executed_tflops": round(exe, 2) if exe else None,
                     "executed_frac": round(exe / peak, 4) if exe else None,
                     "memory_phases": hbm_phases or None,
                     "executed_per_algorithmic": round(executed_tc_flops(cfg, cfg["b"]) / (flops_e * cfg["b"]), 3)
                     if args.engine == "tc" else None},
        "hbm_roofline_edges_per_s": round(pk["hbm_gbs"] * 1e9 / bytes_e, 1),
        "clocks": clk,
    }
    if world == 1 and not args.no_cpu:
        out["cpu_baseline"] = cpu_baseline(W, args, budget_s=args.cpu_seconds)
    return out


# ------------------------------------------------------------------------------ CPU reference path

def batch_list(plan_seq, offsets, p, b):
    """The epoch's batches in plan order: (lo, hi, begin, nb, i, j, bucket_step, batch_in_bucket)."""
    out = []
    for step, (i, j) in enumerate(plan_seq):
        bk = int(i) * p + int(j)
        lo, hi = int(offsets[bk]), int(offsets[bk + 1])
        for k, b0 in enumerate(range(lo, hi, b)):
            out.append((lo, hi, b0 - lo, min(b, hi - b0), int(i), int(j), step, k))
    return out


class CpuTrainer:
    """The reference's CPU training step (oracle/ember_oracle.c orc_train_batch_parts, OpenMP on the host
    cores): per batch sample_negatives -> dedupe of the batch's node ids -> gather of the parameter slice
    -> loss_and_grad -> Adagrad of relations and touched node rows, with partitions i and j held in host
    memory (initialised like the device tables on first use, outside any timed region)."""

    def __init__(self, cfg, edges_fn):
        from oracle import pyoracle as po
        self.po, self.cfg, self.edges_fn = po, cfg, edges_fn
        d = cfg["dim"]
        self.m = po.model(cfg["kind"], dim=d, lr=0.1, eps=1e-10, n_t=cfg["nt"], alpha=cfg["alpha"], chunks=1,
                          seed=NEG_SEED)
        R = cfg["R"] if cfg["kind"] != "dot" else 1
        self.rel_theta = po.init_rows(INIT_SEED ^ 0x52454C, d, 0, R).reshape(R, d)
        self.rel_acc = np.zeros_like(self.rel_theta)
        self.parts = {}

    def part(self, k):
        if k not in self.parts:
            V, p, d = self.cfg["V"], self.cfg["p"], self.cfg["dim"]
            first, rows = self.po.part_offset(V, p, k), self.po.part_size(V, p, k)
            th = self.po.init_rows(INIT_SEED, d, first, rows).reshape(rows, d)
            self.parts[k] = (first, th, np.zeros_like(th))
        return self.parts[k]

    def step(self, batch, epoch=0):
        lo, hi, begin, nb, i, j, step, k = batch
        bucket = self.edges_fn(lo, hi)
        pi, pj = self.part(i), self.part(j)
        return self.po.train_batch_parts(self.m, epoch, step, k, bucket, begin, nb, pi, pj, self.rel_theta,
                                         self.rel_acc)

    def run(self, batches, budget_s, max_steps, threads=None):
        """Timed steps (host wall clock around each C call) until max_steps or budget_s of CPU work."""
        L = self.po.lib()
        all_threads = L.orc_num_threads()
        if threads:
            L.orc_set_num_threads(threads)
        done, t_total, n = 0, 0.0, 0
        try:
            for bt in batches:
                if n >= max_steps or (t_total >= budget_s and n > 0):
                    break
                self.part(bt[4]), self.part(bt[5])  # (table initialisation stays outside the timing)
                t0 = time.perf_counter()
                loss, _ = self.step(bt)
                t_total += time.perf_counter() - t0
                if not np.isfinite(loss):
                    raise RuntimeError("CPU reference: non-finite loss")
                done += bt[3]
                n += 1
            used = L.orc_num_threads()
        finally:
            if threads:
                L.orc_set_num_threads(all_threads)
        return done, t_total, n, used


def cpu_baseline(W, args, budget_s=20.0):
    """The reference CPU path timed on this host beside the GPU run (rank 0, N=1): the same batches as
    the timed GPU steps, full b positives each (sampling and dedupe inside the timing)."""
    cfg = W.cfg
    edges_fn = lambda lo, hi: W.edges[lo:hi].cpu().numpy().view(np.uint32)  # noqa: E731
    start = len(W.batches) // 3 + args.warmup
    cpu = CpuTrainer(cfg, edges_fn)
    done, t, n, thr = cpu.run(W.batches[start:], budget_s, 1000)
    # the 1-thread rate beside the all-core one (one batch of the same stream)
    rest = W.batches[start + n:] or W.batches[start:]  # (small configs: the stream may be used up)
    d1, t1, n1, _ = cpu.run(rest, budget_s / 4, 1, threads=1)
    return {"value": round(done / t, 1), "unit": "edges/s", "cores": thr, "kind": "port",
            "single_thread_value": round(d1 / t1, 1) if t1 > 0 else None,
            "sample": f"{n} full batches (b={cfg['b']} positives, {cfg['nt']}-per-side shared negatives) of the timed "
                      f"GPU steps' batch stream, sampling + dedupe + gather + loss_and_grad + Adagrad "
                      f"(oracle/ember_oracle.c orc_train_batch_parts, OpenMP): {t:.1f} s on {thr} threads "
                      f"(+ {n1} batch, {t1:.1f} s on 1 thread)"}


def bench_reference(args, rank, world):
    """--impl reference: the reference's CPU training step on this host's cores. The reference ships no
    trainer (proj/src/model.cpp, pipeline.cpp absent), so its algorithm runs as our C restatement
    (oracle/ember_oracle.c); the graph comes from the oracle's restatement of the benchmark generator and
    the bucket order from the reference's own make_plan (ordering.cpp built in place, oracle/_ref). Same
    graph, plan, batches (the GPU arm's timed window) and full batch size as our arm; nothing here loads
    the product library."""
    if rank != 0:
        return None
    from oracle import pyoracle as po
    cfg = CONFIGS[args.config]
    t0 = time.perf_counter()
    edges, split = po.graph_generate(cfg["V"], cfg["R"], cfg["E"], GRAPH_SEED, cfg["train"], cfg["valid"])
    bucketed, offsets = po.graph_bucket(cfg["V"], cfg["p"], edges, split, 0)
    del edges, split
    plan = po.ref_plan(0, cfg["p"], cfg["p"], ORDER_SEED)  # OrderingKind::Elimination (ordering.h:14), c = p
    batches = batch_list(plan["seq"], offsets, cfg["p"], cfg["b"])
    setup_s = time.perf_counter() - t0
    cpu = CpuTrainer(cfg, lambda lo, hi: bucketed[lo:hi])
    first = len(batches) // 3 + args.warmup  # the first batch the GPU arm times
    warm = min(args.warmup, 3)  # (untimed, on the batches just before it)
    cpu.run(batches[first - warm:first], 1e9, warm)
    done, t, n, thr = cpu.run(batches[first:], args.cpu_budget, args.steps)
    v = done / t
    return {"metric": METRIC if args.config == "fb86m" else f"train edges/sec ({cfg['desc']})", "impl": "reference",
            "value": round(v, 1), "unit": "edges/s", "n_gpus": world, "steps": n, "warmup": warm,
            "ms_per_step": round(1e3 * t / max(1, n), 3), "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic (same generator, graph, plan and batch stream)",
            "config": {"workload": cfg["desc"], "nodes": cfg["V"], "relations": cfg["R"], "edges_total": cfg["E"],
                       "train_edges": int(offsets[-1]), "model": cfg["kind"], "dim": cfg["dim"], "batch": cfg["b"],
                       "negatives_per_side": cfg["nt"], "alpha": cfg["alpha"], "partitions": cfg["p"],
                       "ordering": "elimination (BETA), reference make_plan", "first_batch": first,
                       "setup_s": round(setup_s, 1)},
            "cpu_baseline": {"value": round(v, 1), "unit": "edges/s", "cores": thr, "kind": "port",
                             "sample": f"{n} full batches of b={cfg['b']} from the GPU arm's timed window (batch "
                                       f"{first} on), sampling + dedupe + gather + loss_and_grad + Adagrad per "
                                       f"step; the reference has no runnable trainer (proj/src/model.cpp absent), "
                                       f"oracle/ember_oracle.c is its SPEC restatement"
                                       + (f"; stopped at the {args.cpu_budget:.0f} s budget" if n < args.steps else "")},
            "e2e": {"value": round(v, 1), "unit": "edges/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "native_libraries": loaded_native_libraries()}


def loaded_native_libraries():
    """The repo's own shared objects mapped into this process (the reference arm must map only oracle/)."""
    libs = set()
    try:
        for line in open("/proc/self/maps"):
            path = line.split()[-1] if len(line.split()) >= 6 else ""
            if path.startswith(ROOT) and path.endswith(".so"):
                libs.add(os.path.relpath(path, ROOT))
    except OSError:
        pass
    return sorted(libs)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="fb86m", choices=sorted(CONFIGS))
    ap.add_argument("--engine", default=os.environ.get("EMBER_ENGINE", "tc"), choices=["simt", "tc"])
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    ap.add_argument("--cpu-budget", type=float, default=150.0,
                    help="--impl reference: stop timing after this many seconds of CPU work")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--capacity", type=int, default=0,
                    help="partition-buffer capacity c < p: train through the device buffer (one timed epoch)")
    ap.add_argument("--distributed", action="store_true",
                    help="use the multi-GPU round-schedule path even at N=1 (a 1-rank NCCL group; for checks)")
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)
    if args.engine == "simt":  # the fp32 reference engine (baseline measurements only)
        os.environ["EMBER_TEST_ENGINES"] = "1"
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    # stdout carries exactly one JSON line: native libraries' banners (e.g. NCCL's version line at
    # communicator creation) go to stderr until the result is printed
    sys.stdout.flush()
    saved_stdout = os.dup(1)
    os.dup2(2, 1)
    try:
        out = _run(args, rank, world, local_rank)
    finally:
        sys.stdout.flush()
        os.dup2(saved_stdout, 1)
        os.close(saved_stdout)
    if out is not None:
        print(json.dumps(out), flush=True)


def _run(args, rank, world, local_rank):
    out = None
    if args.impl == "reference":
        out = bench_reference(args, rank, world)
    else:
        dist_path = world > 1 or args.distributed
        if dist_path:
            import torch
            import torch.distributed as dist
            local_rank %= max(1, torch.cuda.device_count())  # (more ranks than GPUs: gloo checks only)
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            os.environ.setdefault("MASTER_PORT", "29533")
            os.environ.setdefault("RANK", str(rank))
            os.environ.setdefault("WORLD_SIZE", str(world))
            torch.cuda.set_device(local_rank)
            backend = os.environ.get("EMBER_DIST_BACKEND", "nccl")  # gloo: multi-rank checks on one GPU
            dist.init_process_group(backend, device_id=torch.device(f"cuda:{local_rank}") if backend == "nccl" else None)
        if dist_path:
            out = bench_distributed(args, rank, world, local_rank)
        elif args.capacity:
            out = bench_buffered(args, local_rank)
        else:
            out = bench_ours(args, rank, world, local_rank)
        if dist_path:
            import torch.distributed as dist
            dist.destroy_process_group()
    return out


if __name__ == "__main__":
    main()
