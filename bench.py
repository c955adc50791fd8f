#!/usr/bin/env python
"""Lattice hot-path benchmark (BASELINE.json metric: Lattice Network samples/sec).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload micro|mid] [--impl ours|reference]

One process per GPU (torchrun for N > 1, NCCL barrier, max-over-ranks device time).
Workloads:
  micro -- embedding-bag microbench: 64 tables x 1M rows x 128, B=16384, bags U[0,40]
  mid   -- mid Lattice Network, bf16, B=32768 per GPU (default once the network is built)
A "step" is one pass of the hot path over one batch of synthetic input already resident in
HBM (`value`); `e2e` repeats it through the public C-ABI call with the batch's inputs copied
from pinned host memory and the result copied back inside the timed region.
`--impl reference` times the CPU oracle port of the same workload on the host's cores
(rank 0 only; the reference has no implementation of the network).
"""
import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

SEED_T, SEED_D = 0x1A77, 0x1A78


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return p["hbm_gbs"], p["bf16_tflops"], p.get("bf16_tflops_sustained", p["bf16_tflops"]), "measured"
    except Exception:
        return 6650.0, 1590.0, 1400.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    def __init__(self, index):
        self.index = index
        self.samples = []
        self.proc = None

    def __enter__(self):
        self.t_start = None
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
            time.sleep(1.0)  # nvidia-smi start-up must not overlap the timed region
        except Exception:
            self.proc = None
        return self

    def mark(self):
        """Start of the timed region: samples before it are discarded."""
        self.t_start = time.time()

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 7 and self.t_start is not None and time.time() >= self.t_start:
                self.samples.append(parts)

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4) if s[3 + i] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.samples)}


def dist_setup(n):
    import torch
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        torch.cuda.set_device(0)
    return rank, world, local


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def max_over_ranks(x, world):
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


# ------------------------------------------------------------------------------------------------
# micro: embedding-bag microbench (configs[1])
# ------------------------------------------------------------------------------------------------
MICRO = dict(F=64, rows=1_000_000, D=128, B=16384, max_len=40)


def micro_bytes(n_ids, F, B, D, s_tab, s_out):
    return n_ids * D * s_tab + n_ids * 4 + (F * B + 1) * 8 + F * B * D * s_out


def run_micro(args, rank, world, local):
    import torch
    import paper_2512_09200_b200 as L
    c = MICRO
    F, R, D, B, ML = c["F"], c["rows"], c["D"], c["B"], c["max_len"]
    dt = torch.bfloat16 if args.dtype == "bf16" else torch.float32
    s_tab = 2 if dt == torch.bfloat16 else 4
    tab = torch.empty((F, R, D), dtype=dt, device="cuda")
    L.fill_tables(tab, SEED_T)
    tables = list(tab.unbind(0))
    ptrs = torch.tensor([t.data_ptr() for t in tables], dtype=torch.int64, device="cuda")
    rows = torch.full((F,), R, dtype=torch.int64, device="cuda")
    # per-rank distinct batches (weak scaling: every rank processes its own B samples)
    offsets, ids = L.synth_bags(F, B, ML, R, SEED_D + rank)
    n_ids = int(offsets[-1].item())
    out = torch.empty((B, F, D), dtype=dt, device="cuda")
    stream = torch.cuda.current_stream()

    def step():
        L.embedding_bag(tables, offsets, ids, B, out=out, check_errors=False, table_ptrs=ptrs,
                        rows=rows)

    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    kev = [torch.cuda.Event(enable_timing=True) for _ in range(2 * args.steps)]
    with ClockSampler(local) as clk:
        for _ in range(args.warmup):
            step()
        torch.cuda.synchronize()
        barrier(world)
        torch.cuda.synchronize()
        clk.mark()
        ev0.record(stream)
        for i in range(args.steps):
            kev[2 * i].record(stream)
            step()
            kev[2 * i + 1].record(stream)
        ev1.record(stream)
        torch.cuda.synchronize()
    barrier(world)
    torch.cuda.synchronize()
    ms = max_over_ranks(ev0.elapsed_time(ev1) / args.steps, world)
    kms = [kev[2 * i].elapsed_time(kev[2 * i + 1]) for i in range(args.steps)]
    value = world * B / (ms / 1e3)

    # e2e through the public call with host buffers: H2D offsets+ids, D2H pooled output
    h_off = offsets.cpu().pin_memory()
    h_ids = ids[:n_ids].cpu().pin_memory()
    d_off = torch.empty_like(offsets)
    d_ids = torch.empty(n_ids, dtype=torch.int32, device="cuda")
    h_out = torch.empty(out.shape, dtype=dt, pin_memory=True)

    def e2e_step():
        d_off.copy_(h_off, non_blocking=True)
        d_ids.copy_(h_ids, non_blocking=True)
        L.embedding_bag(tables, d_off, d_ids, B, out=out, check_errors=False, table_ptrs=ptrs,
                        rows=rows)
        h_out.copy_(out, non_blocking=True)

    for _ in range(2):
        e2e_step()
    torch.cuda.synchronize()
    barrier(world)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        e2e_step()
    e1.record(stream)
    torch.cuda.synchronize()
    e2e_ms = max_over_ranks(e0.elapsed_time(e1) / args.steps, world)

    hbm, _, _, src = load_peaks()
    alg = micro_bytes(n_ids, F, B, D, s_tab, s_tab)
    kernel_ms = statistics.mean(kms)
    achieved = alg / (kernel_ms / 1e3) / 1e9
    res = {
        "metric": "embedding-bag samples/sec (configs[1] microbench)",
        "value": value, "unit": "samples/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32" if s_tab == 4 else "bf16", "data": "synthetic",
        "config": {"workload": "micro: 64 tables x 1M rows x 128, B=16384/GPU, bags U[0,40]",
                   "tables_gb": F * R * D * s_tab / 1e9, "ids_per_step": n_ids,
                   "l2": "inputs larger than L2 (uniform random rows over %.1f GB)" % (F * R * D * s_tab / 1e9),
                   "parallelism": f"replicas x{world}"},
        "e2e": {"value": world * B / (e2e_ms / 1e3), "unit": "samples/s",
                "h2d_bytes_per_step": (F * B + 1) * 8 + n_ids * 4,
                "d2h_bytes_per_step": B * F * D * s_tab},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s",
                     "frac": achieved / hbm, "traffic": None, "kernel": "bag_kernel",
                     "peak_source": src, "algorithmic_bytes_per_launch": alg,
                     "kernel_ms_mean": kernel_ms, "kernel_ms_min": min(kms), "kernel_ms_max": max(kms)},
        "gpu_launches": args.steps,
        "clocks": clk.summary(),
    }
    return res, dict(F=F, R=R, D=D, B=B, ML=ML, offsets=offsets, ids=ids)


def cpu_baseline_micro(seconds=15.0):
    """Oracle (port) embedding bag on a bounded sample, all host threads."""
    import numpy as np
    import oracle
    c = MICRO
    F, R, D, B, ML = c["F"], c["rows"], c["D"], c["B"], c["max_len"]
    threads = os.cpu_count() or 1
    o, i = oracle.synth_bags(F, B, ML, R, SEED_D)
    n, t0 = 0, time.perf_counter()
    chunk = 64
    while time.perf_counter() - t0 < seconds and n + chunk <= B:
        oracle.embedding_bag_synth(SEED_T, F, R, D, B, o, i, n, n + chunk, threads)
        n += chunk
    dt = time.perf_counter() - t0
    return {"value": n / dt, "unit": "samples/s", "cores": threads, "kind": "port",
            "sample": f"{n} of {B} samples of the micro batch ({dt:.1f} s, tables regenerated lazily)"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--workload", default="micro", choices=["micro"])
    ap.add_argument("--dtype", default="f32", choices=["f32", "bf16"])
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    if args.impl == "reference":
        rank = int(os.environ.get("RANK", "0"))
        if rank != 0:
            return
        steps = []
        for _ in range(args.warmup + args.steps):
            steps.append(cpu_baseline_micro(seconds=max(2.0, args.cpu_seconds / max(args.steps, 1))))
        vals = [s["value"] for s in steps[args.warmup:]]
        v = statistics.median(vals)
        cb = dict(steps[-1])
        cb["value"] = v
        print(json.dumps({"impl": "reference", "metric": "embedding-bag samples/sec (configs[1] microbench)",
                          "value": v, "unit": "samples/s", "n_gpus": 0, "steps": args.steps,
                          "warmup": args.warmup, "higher_is_better": True,
                          "config": {"workload": "micro: 64 tables x 1M rows x 128, B=16384, bags U[0,40]"},
                          "dtype": "f32", "data": "synthetic", "cpu_baseline": cb,
                          "e2e": {"value": v, "unit": "samples/s", "h2d_bytes_per_step": 0,
                                  "d2h_bytes_per_step": 0}}))
        return

    rank, world, local = dist_setup(args.gpus)
    res, _ = run_micro(args, rank, world, local)
    if rank == 0:
        if world == 1:
            res["cpu_baseline"] = cpu_baseline_micro(args.cpu_seconds)
        print(json.dumps(res))
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
