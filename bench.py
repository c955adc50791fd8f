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


def load_traffic(workload, kernel, key="dram"):
    """Bytes per launch (group) of `kernel` from the committed ncu captures (profiles/r02, else
    r01): key "dram" = dram__bytes_read.sum + dram__bytes_write.sum, "l2" = lts__t_bytes.sum."""
    for rnd in ("r02", "r01"):
        try:
            with open(os.path.join(ROOT, "profiles", rnd, "traffic.json")) as f:
                v = json.load(f).get(workload, {}).get(kernel)
        except Exception:
            continue
        if isinstance(v, dict):
            v = v.get(key)
        elif key != "dram":
            v = None
        if v is not None:
            return v
    return None


def load_l2_peak():
    """Measured L2 read bandwidth (GB/s, scripts/l2_probe.cu on a B200: profiles/r02/l2_probe.json)."""
    try:
        with open(os.path.join(ROOT, "profiles", "r02", "l2_probe.json")) as f:
            return json.load(f)["l2_read_gbs"]
    except Exception:
        return None


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
                                          "--format=csv,noheader,nounits", "-lms", "50"],
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
            # a line read within 20 ms of the mark may have been sampled before it
            if len(parts) >= 7 and self.t_start is not None and time.time() >= self.t_start + 0.02:
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


def run_micro(args, rank, world, local, dtype=None, min_seconds=0.0):
    import torch
    import paper_2512_09200_b200 as L
    c = MICRO
    F, R, D, B, ML = c["F"], c["rows"], c["D"], c["B"], c["max_len"]
    dt = torch.bfloat16 if (dtype or args.dtype) == "bf16" else torch.float32
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
    steps = args.steps
    if min_seconds > 0:  # long enough a timed region for the clock sampler to see it
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        step()
        e0.record(stream)
        for _ in range(3):
            step()
        e1.record(stream)
        torch.cuda.synchronize()
        steps = max(steps, int(min_seconds * 1e3 / (e0.elapsed_time(e1) / 3)) + 1)
    args = argparse.Namespace(**dict(vars(args), steps=steps))
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
                     "frac": achieved / hbm,
                     "traffic": load_traffic("micro_bf16" if dt == torch.bfloat16 else "micro_f32", "bag_kernel"),
                     "kernel": "bag_kernel",
                     "peak_source": src, "algorithmic_bytes_per_launch": alg,
                     "kernel_ms_mean": kernel_ms, "kernel_ms_min": min(kms), "kernel_ms_max": max(kms)},
        "gpu_launches": args.steps,
        "clocks": clk.summary(),
    }
    return res, dict(F=F, R=R, D=D, B=B, ML=ML, offsets=offsets, ids=ids)


def cpu_baseline_micro(seconds=15.0, threads=None):
    """Oracle (port) embedding bag on a bounded sample (all host threads unless given)."""
    import numpy as np
    import oracle
    c = MICRO
    F, R, D, B, ML = c["F"], c["rows"], c["D"], c["B"], c["max_len"]
    threads = threads or os.cpu_count() or 1
    o, i = oracle.synth_bags(F, B, ML, R, SEED_D)
    n, t0 = 0, time.perf_counter()
    chunk = 64
    while time.perf_counter() - t0 < seconds and n + chunk <= B:
        oracle.embedding_bag_synth(SEED_T, F, R, D, B, o, i, n, n + chunk, threads)
        n += chunk
    dt = time.perf_counter() - t0
    return {"value": n / dt, "unit": "samples/s", "cores": threads, "kind": "port",
            "sample": f"{n} of {B} samples of the micro batch ({dt:.1f} s, tables regenerated lazily)"}


# ------------------------------------------------------------------------------------------------
# mid: the Lattice Network step (configs[2]); builder widths from SURVEY.md 8d
# ------------------------------------------------------------------------------------------------
MID = dict(n=256, d=128, blocks=4, nF=128, nL=128, k=32, mlp=[8192, 2048, 2048, 16384],
           domains=4, heads=6, tower_hidden=512)
MID_ROWS, MID_B, MID_MAXLEN = 100_000, 32768, 40
SEED_W = 0x1A79


def dense_flops_per_sample(c):
    n, d, k, nL = c["n"], c["d"], c["k"], c["nL"]
    mlp = c["mlp"]
    per_block = 4 * n * d * k + 2 * nL * n * d + 2 * sum(mlp[i] * mlp[i + 1] for i in range(len(mlp) - 1))
    dense = 2 * (c.get("dense_in", 0) * c.get("dense_hidden", 0) +
                 c.get("dense_hidden", 0) * c.get("dense_features", 0) * d)  # dense processor
    return c["blocks"] * per_block + 2 * (n * d * c["tower_hidden"] + c["tower_hidden"] * c["heads"]) + dense


def mlp_flops_per_sample(c):
    mlp = c["mlp"]
    return 2 * sum(mlp[i] * mlp[i + 1] for i in range(len(mlp) - 1))


FULL_TASKS, FULL_WINDOWS = 4, [5400000, 86400000, 604800000]  # O = 4 objectives, {90min, 1d, 7d}
FULL_DENSE = (16, 64, 256)  # dense embeddings, dense processor input width, dense processor hidden
FULL_MERGED, FULL_TEACHER = 48, 16  # union-schema width of the merged dense features, KTAP teacher dim
FULL_STORE, FULL_TTL = 1 << 20, 4 * 3600 * 1000  # KTAP teacher store entries, TTL (ms)


LARGE = dict(n=512, d=128, blocks=4, nF=256, nL=256, k=32, mlp=[16384, 2048, 2048, 32768],
             domains=4, heads=6, tower_hidden=512)
LARGE_ROWS, LARGE_B = 1_500_000, 65536  # 512 x 1.5M x 128 bf16 = 196.6 GB: needs >= 2 GPUs


def run_mid(args, rank, world, local):
    import torch
    import paper_2512_09200_b200 as L
    full = args.workload == "full"
    large = args.workload == "large"
    global MID_ROWS, MID_B
    if large:  # configs[3]: table-wise sharded over >= 2 GPUs, B = 64k per GPU
        if world < 2:
            raise SystemExit("--workload large needs >= 2 GPUs (196 GB of tables)")
        MID_ROWS, MID_B = LARGE_ROWS, LARGE_B
    # full consolidated portfolio: 16 domains, heads = 4 objectives x 3 attribution windows,
    # Zipper window assignment + window-routed heads in every step (mid-width backbone)
    if full and world > 1:  # configs[4] on >= 2 GPUs: the large backbone, table-wise sharded
        large = True
        MID_ROWS, MID_B = LARGE_ROWS, LARGE_B
    backbone = LARGE if large else MID
    c = dict(backbone, domains=16, heads=FULL_TASKS * len(FULL_WINDOWS), dense_features=FULL_DENSE[0],
             dense_in=FULL_DENSE[1], dense_hidden=FULL_DENSE[2]) if full else backbone
    n, d, B = c["n"], c["d"], MID_B
    nc = n - c.get("dense_features", 0)  # embeddings pooled from tables (the rest: dense processor)
    net = L.Network(**c, max_batch=B, weight_seed=SEED_W)
    sharded = world > 1 or args.exchange == "peer1"  # peer1: the peer path at N=1 (experiments)
    peer = sharded and args.exchange in ("peer", "peer1")
    if sharded:  # table-wise: this rank owns features [rank*n/W, (rank+1)*n/W)
        from paper_2512_09200_b200.sharded import ShardedBags
        sb = ShardedBags(nc, B, d, world, rank)
        n_tab = sb.Fl
        tab = torch.empty((n_tab, MID_ROWS, d), dtype=torch.bfloat16, device="cuda")
        L.fill_tables(tab, SEED_T, feature_base=sb.owned()[0], rows_total=MID_ROWS)
        if peer:  # owners write pooled rows straight into every rank's X0 over NVLink
            from paper_2512_09200_b200.peer import PeerBags
            pb = PeerBags(net, nc, B, d, world, rank, row_stride=n * d)
        else:
            send = torch.empty((world * B, sb.Fl, d), dtype=torch.bfloat16, device="cuda")
            recv = torch.empty_like(send)
    else:
        n_tab = nc
        tab = torch.empty((nc, MID_ROWS, d), dtype=torch.bfloat16, device="cuda")
        L.fill_tables(tab, SEED_T)
    tables = list(tab.unbind(0))
    ptrs = torch.tensor([t.data_ptr() for t in tables], dtype=torch.int64, device="cuda")
    rows = torch.full((n_tab,), MID_ROWS, dtype=torch.int64, device="cuda")
    offsets, ids = L.synth_bags(nc, B, MID_MAXLEN, MID_ROWS, SEED_D + rank)
    dom = L.synth_domains(B, c["domains"], SEED_D + rank)
    n_ids = int(offsets[-1].item())
    if peer:
        pb.register("main", offsets, ids)
    elif sharded:  # static exchange capacity (setup, outside the timed region): max slice over ranks
        import torch.distributed as dist
        cnt, _ = sb.slice_counts(offsets)
        cap = cnt.max().reshape(1)
        dist.all_reduce(cap, op=dist.ReduceOp.MAX)
        sb.capacity = int(cap.item())
    logits = torch.empty((B, c["heads"]), dtype=torch.float32, device="cuda")
    stream = torch.cuda.current_stream()
    key_of = {id(offsets): "main"}  # peer exchange: input buffer pair -> registered key

    if full:
        imp = L.synth_impressions(B, FULL_TASKS, 7 + rank)
        # dense features of the 16 consolidated domains: domain g declares its own subset of a
        # 64-name pool; merge_domains re-lays them out under the union schema every step
        g_dense = torch.Generator().manual_seed(0xD15E)
        declared = [[f"x{int(i)}" for i in torch.randperm(FULL_MERGED, generator=g_dense)[:8 + 2 * g]]
                    for g in range(c["domains"])]
        union, src = L.union_schema(declared)
        src_col = torch.full((c["domains"], FULL_MERGED), -1, dtype=torch.int32)
        src_col[:, : len(union)] = torch.tensor(src, dtype=torch.int32)
        src_col = src_col.cuda()
        max_decl = max(len(x) for x in declared)
        dvals = torch.randn((B, max_decl), generator=torch.Generator(device="cuda").manual_seed(rank),
                            device="cuda")
        # KTAP teacher store: 1M precomputed teacher embeddings with write times;
        # each sample's (user, ad) pair maps to an entry (25% never computed), ~1/3 expired
        gk = torch.Generator(device="cuda").manual_seed(0x7EAC + rank)
        store_emb = torch.randn((FULL_STORE, FULL_TEACHER), generator=gk, device="cuda")
        store_logit = torch.randn(FULL_STORE, generator=gk, device="cuda")
        t_now = 1_700_000_000_000
        written_at = t_now - torch.randint(0, FULL_TTL * 3 // 2, (FULL_STORE,), generator=gk, device="cuda")
        slot = torch.randint(0, FULL_STORE, (B,), generator=gk, device="cuda")
        slot[torch.rand(B, generator=gk, device="cuda") < 0.25] = -1
        nW = len(FULL_WINDOWS)
        obj_out = (torch.empty((B, FULL_TASKS), dtype=torch.float32, device="cuda"),
                   torch.empty(FULL_TASKS, dtype=torch.float64, device="cuda"),
                   torch.empty(nW, dtype=torch.int64, device="cuda"),
                   torch.empty((nW, FULL_TASKS), dtype=torch.int64, device="cuda"))
        wp = [1.0 / len(FULL_WINDOWS)] * len(FULL_WINDOWS)

    def forward(dm, off, ii, out, imp_cols=None, dv=None):
        dense = None
        if full:  # K5: window assignment + per-window labels of this batch's impressions
            win, lab, _ = L.zipper_assign_labels(*(imp_cols or imp), FULL_WINDOWS, wp, 7, routed=False,
                                               check_errors=False)
            # merge_domains (union schema, zero padding), then KTAP student inputs [merged dense ||
            # clipped teacher embedding or zeros] -> the dense processor's input
            dv_, slot_ = dv if dv is not None else (dvals, slot)
            merged = L.merge_dense(dm, dv_, src_col, FULL_MERGED, out_dtype=torch.float32, check_errors=False)
            dense, _, _ = L.student_inputs(merged, slot_, store_emb, written_at, FULL_TTL, t_now,
                                           store_logit=store_logit, clip=3.0, smoothing=0.1)
        if peer:
            pb.forward(key_of[id(off)], dm, tables, ptrs, rows, logits=out, dense=dense)
        elif sharded:
            pooled = sb.forward_embeddings(off, ii, tables, ptrs, rows, send=send, recv=recv)
            net.forward(dm, pooled=pooled, shards=world, logits=out, dense=dense)
        else:
            net.forward(dm, off, ii, ptrs, rows, torch.bfloat16, logits=out, dense=dense)
        if full:  # the window mask applied to the heads (training routes each sample's loss)
            # post-tower batch step: routed logits, per-task correlation loss (fp64), window summary
            L.routed_objectives(out, win, lab, FULL_TASKS, nW, check_errors=False, out=obj_out)

    def step():
        forward(dom, offsets, ids, logits)

    step_eager = step
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        for _ in range(args.warmup):
            step()
        torch.cuda.synchronize()
        if args.graph:  # the whole forward step captured once and replayed (no per-kernel host launches)
            graph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(graph):
                forward(dom, offsets, ids, logits)
            stream = torch.cuda.current_stream()
            graph.replay()
            torch.cuda.synchronize()
            step = graph.replay
        barrier(world)
        torch.cuda.synchronize()
        clk.mark()
        ev0.record(stream)
        for _ in range(args.steps):
            step()
        ev1.record(stream)
        torch.cuda.synchronize()
    barrier(world)
    torch.cuda.synchronize()
    ms = max_over_ranks(ev0.elapsed_time(ev1) / args.steps, world)
    value = world * B / (ms / 1e3)

    # per-stage device times (separate pass, events between stages)
    net.set_timing(True)
    stages, emb_ms, peer_split = [], [], []
    dense0 = L.student_inputs(L.merge_dense(dom, dvals, src_col, FULL_MERGED, out_dtype=torch.float32), slot,
                              store_emb, written_at, FULL_TTL, t_now)[0] if full else None
    for _ in range(5):
        if peer:  # bucket + barrier + owner kernel (NVLink reads/stores) + barrier
            barrier(world)
            a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a0.record(stream)
            pb.forward_embeddings("main", dom, tables, ptrs, rows, timed=True)
            a1.record(stream)
            net.forward_in_place(dom, logits=logits, dense=dense0)
            torch.cuda.synchronize()
            emb_ms.append(a0.elapsed_time(a1))
            peer_split.append(pb.stage_ms())
        elif sharded:  # ids a2a + owner pooling + pooled a2a, timed on the stream
            a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a0.record(stream)
            pooled = sb.forward_embeddings(offsets, ids, tables, ptrs, rows, send=send, recv=recv)
            a1.record(stream)
            net.forward(dom, pooled=pooled, shards=world, logits=logits, dense=dense0)
            torch.cuda.synchronize()
            emb_ms.append(a0.elapsed_time(a1))
        else:
            step_eager()
        stages.append(net.stage_times())
    net.set_timing(False)
    st = [statistics.median(s[i] for s in stages) for i in range(len(stages[0]))]
    # stages: [bucket, bag (or shard gather), (fm_lcb, mlp) x blocks, tower]
    t_bag = st[1] + (min(emb_ms) if sharded else 0.0)
    t_fm = [st[2 + 2 * b] for b in range(c["blocks"])]
    t_mlp = [st[3 + 2 * b] for b in range(c["blocks"])]
    t_tower = st[2 + 2 * c["blocks"]]
    hbm, tf_burst, tf_sust, src = load_peaks()
    emb_bytes = micro_bytes(n_ids, nc, B, d, 2, 2)
    flops = dense_flops_per_sample(c) * B
    mlp_fl = mlp_flops_per_sample(c) * B
    mlp_ms = statistics.mean(t_mlp)
    mlp_achieved = mlp_fl / (mlp_ms / 1e3) / 1e12
    dense_ms = sum(t_fm) + sum(t_mlp) + t_tower
    fm_bytes = B * (n * d * 2 + n * c["k"] * 2 + c["nL"] * d * 2)

    # e2e through the public call: pinned-host sparse batch -> H2D (copy stream, double
    # buffered) -> forward -> D2H logits, every step inside the timed region
    h_off = offsets.cpu().pin_memory()
    h_ids = ids[:n_ids].cpu().pin_memory()
    h_dom = dom.cpu().pin_memory()
    h_out = torch.empty((B, c["heads"]), dtype=torch.float32, pin_memory=True)
    bufs = [(torch.empty_like(offsets), torch.empty(n_ids, dtype=torch.int32, device="cuda"),
             torch.empty_like(dom)) for _ in range(2)]
    if peer:  # the double-buffered H2D destinations are published to the owners once
        for i, (o, ii, _) in enumerate(bufs):
            pb.register(i, o, ii)
            key_of[id(o)] = i
    if full:  # the impression log columns travel with the batch too
        h_imp = [t.cpu().pin_memory() for t in imp]
        d_imp = [[torch.empty_like(t) for t in imp] for _ in range(2)]
        h_dv = (dvals.cpu().pin_memory(), slot.cpu().pin_memory())  # per-step dense values + KTAP slots
        d_dv = [(torch.empty_like(dvals), torch.empty_like(slot)) for _ in range(2)]
    cstream = torch.cuda.Stream()
    copied = [torch.cuda.Event() for _ in range(2)]
    consumed = [torch.cuda.Event() for _ in range(2)]

    def h2d(i):
        o, ii, dm = bufs[i % 2]
        with torch.cuda.stream(cstream):
            cstream.wait_event(consumed[i % 2])
            o.copy_(h_off, non_blocking=True)
            ii.copy_(h_ids, non_blocking=True)
            dm.copy_(h_dom, non_blocking=True)
            if full:
                for dst, src in zip(d_imp[i % 2], h_imp):
                    dst.copy_(src, non_blocking=True)
                for dst, src in zip(d_dv[i % 2], h_dv):
                    dst.copy_(src, non_blocking=True)
            copied[i % 2].record(cstream)

    e2e_graphs = [None, None]  # the forward over each input buffer, replayed like the device-resident step

    def e2e_forward(i):
        if e2e_graphs[i % 2] is not None:
            e2e_graphs[i % 2].replay()
            return
        o, ii, dm = bufs[i % 2]
        forward(dm, o, ii, logits, d_imp[i % 2] if full else None, d_dv[i % 2] if full else None)

    def e2e_run(k):
        for e in consumed:
            e.record(stream)
        h2d(0)
        for i in range(k):
            if i + 1 < k:
                h2d(i + 1)
            stream.wait_event(copied[i % 2])
            e2e_forward(i)
            consumed[i % 2].record(stream)
            h_out.copy_(logits, non_blocking=True)

    e2e_run(2)
    torch.cuda.synchronize()
    if args.graph:  # the same launch path as `value`: the forward step of each buffer from a graph
        for i in range(2):
            g = torch.cuda.CUDAGraph()
            o, ii, dm = bufs[i]
            with torch.cuda.graph(g):
                forward(dm, o, ii, logits, d_imp[i] if full else None, d_dv[i] if full else None)
            e2e_graphs[i] = g
        stream = torch.cuda.current_stream()
        e2e_run(2)
        torch.cuda.synchronize()
    barrier(world)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    e2e_run(args.steps)
    e1.record(stream)
    torch.cuda.synchronize()
    e2e_ms = max_over_ranks(e0.elapsed_time(e1) / args.steps, world)

    # per step: domain bucketing (histogram, block scan, ranks) + tiles + bag, then per block the
    # FM/LCB kernel and one GEMM per MLP layer, then the grouped tower
    launches = 5 + c["blocks"] * (1 + len(c["mlp"]) - 1) + 1
    if os.environ.get("LATTICE_TOWER_PAIR", "1") != "0":
        launches += 1  # the towers run as the CTA-pair swish GEMM + tower_heads_kernel
    if peer:
        pb.check()
        launches += 2  # two barrier kernels (the bag slot above is the owner kernel)
    elif sharded:
        sb.check_overflow()
        launches += 2  # owner bag kernel + offsets scan (the bag slot above is the shard gather)
    if full:
        launches += 6  # zipper_kernel + summary + 2 x (moments + fold) of routed_objectives
        launches += 5  # merge_dense + student_inputs + 2 dense GEMMs + dense row norm
    if full:
        metric = "Lattice Network samples/sec (full consolidated portfolio, forward step)"
        wl = ("full consolidated portfolio: 16 domains x (4 objectives x 3 windows {90min,1d,7d}) "
              "heads, per-sample Zipper window assignment (seed 7, p=1/3) + window-routed heads + correlation loss + window summary each step; 16 dense embeddings from a "
              "dense processor over [48-wide union schema of the domains' dense features (merge_domains "
              "zero padding) || KTAP teacher embedding (16, 1M-entry store, TTL 4h, clipped; zeros on "
              "miss)], MLP 64-256-16x128, in place of 16 tables; "
              + ("large backbone (512 tables x 1.5M rows x 128 bf16 = 196.6 GB table-wise sharded, l=4, "
                 "n=512, MLP 16384-2048-2048-32768, tower 65536-512-12), B=65536/GPU" if large else
                 "mid-width backbone on 1 GPU (256 sparse feats x 100k rows x 128, l=4, "
                 "MLP 8192-2048-2048-16384, tower 32768-512-12), B=32768/GPU"))
    elif large:
        metric = "Lattice Network samples/sec (large config, forward step)"
        wl = ("large Lattice Network: 512 tables x 1.5M rows x 128 bf16 (196.6 GB) table-wise sharded, "
              "l=4 DWFB blocks (n=512, nF=nL=256, k=32, MLP 16384-2048-2048-32768), 4 domains x 6 heads, "
              "tower 65536-512-6, B=65536/GPU")
    else:
        metric = "Lattice Network samples/sec (mid config, forward step)"
        wl = ("mid Lattice Network: 256 sparse feats x 100k rows x 128, l=4 DWFB blocks (nF=nL=128, k=32, "
              "MLP 8192-2048-2048-16384), 4 domains x 6 heads, tower 32768-512-6, B=32768/GPU")
    res = {
        "metric": metric,
        "value": value, "unit": "samples/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "bf16", "data": "synthetic (counter-based tables/bags/weights)",
        "config": {"workload": wl,
                   "global_batch": world * B, "ids_per_step": n_ids,
                   "l2": ("embedding rows drawn uniformly from %.1f GB of tables per GPU; activations %.1f GB/buffer (> L2)"
                          % (n_tab * MID_ROWS * d * 2 / 1e9, B * n * d * 2 / 1e9)),
                   "launch": "CUDA graph replay of the forward step" if args.graph else "eager launches",
                   "parallelism": ((f"table-wise sharded embeddings over {world} GPUs (owner kernel reads "
                                    f"peers' ids and stores pooled rows into their X0 over NVLink via CUDA "
                                    f"IPC, in-kernel barriers, no NCCL on the data path) + dense replicas")
                                   if peer else
                                   (f"table-wise sharded embeddings over {world} GPUs (ids + pooled "
                                    f"all-to-all, NCCL/NVLink) + dense replicas")) if sharded else "1 GPU"},
        "e2e": {"value": world * B / (e2e_ms / 1e3), "unit": "samples/s",
                "h2d_bytes_per_step": (nc * B + 1) * 8 + n_ids * 4 + B * 4 +
                                      (sum(t.numel() * t.element_size() for t in imp) + dvals.numel() * 4 +
                                       slot.numel() * 8 if full else 0),
                "d2h_bytes_per_step": B * c["heads"] * 4},
        "roofline": {"bound": "tensor", "achieved": mlp_achieved, "peak": tf_burst, "unit": "TFLOP/s",
                     "frac": mlp_achieved / tf_burst,
                     "traffic": load_traffic("mid", "gemm_mlp_group") if args.workload == "mid" else None,
                     "kernel": "gemm2_kernel (CTA-pair tcgen05 GEMM; FMB MLP, 3 GEMMs per block, fused swish_rn / "
                               "residual-norm)",
                     "peak_source": f"{src} burst (the conservative denominator: the MLP GEMMs exceed the "
                                    f"measured sustained figure {tf_sust})",
                     "algorithmic_flops_per_launch_group": mlp_fl, "ms": mlp_ms},
        "stages": {
            "_note": ("per-stage CUDA-event times: median of 5 eager forwards with events between "
                      "stages (the graph-replayed step has no events inside)"),
            "embedding": emb_stage(args.workload if not sharded else None, t_bag, emb_bytes, hbm),
            "fm_lcb": {"ms_per_block": statistics.mean(t_fm), "bytes_per_block": fm_bytes,
                       "GB/s": fm_bytes / (statistics.mean(t_fm) / 1e3) / 1e9,
                       "frac_hbm": fm_bytes / (statistics.mean(t_fm) / 1e3) / 1e9 / hbm},
            "mlp": {"ms_per_block": mlp_ms, "TFLOP/s": mlp_achieved, "frac_tensor_sustained": mlp_achieved / tf_sust,
                    "frac_tensor_burst": mlp_achieved / tf_burst},
            "tower": {"ms": t_tower, "TFLOP/s": 2 * B * n * d * c["tower_hidden"] / (t_tower / 1e3) / 1e12},
            "dense_total": {"ms": dense_ms, "TFLOP": flops / 1e12,
                            "TFLOP/s": flops / (dense_ms / 1e3) / 1e12},
            "bucket_ms": st[0],
            # sharded: the embedding exchange runs outside the network's own stage events
            "stage_sum_ms": sum(st) + (min(emb_ms) if sharded else 0.0),
            "eager_vs_graph_ms": sum(st) + (min(emb_ms) if sharded else 0.0) - ms,
        },
        "gpu_launches": launches * args.steps,
        "clocks": clk.summary(),
    }
    if peer:  # embedding stage split on rank 0: [bucket, barrier 1, owner kernel, barrier 2] ms
        res["stages"]["embedding"]["peer_split_ms"] = [min(x[i] for x in peer_split) for i in range(4)]
    return res


def emb_stage(workload, t_ms, alg_bytes, hbm):
    """Embedding-stage roofline. The algorithmic bytes (every gathered row counted once per id,
    SURVEY 8d emb_bytes) exceed what DRAM serves: the mid tables (25.6 MB each, visited table by
    table) stay hot in L2, so the line also carries the ncu-measured DRAM and L2 bytes of the bag
    kernel at this config (profiles/r02/traffic.json) against the HBM and measured L2 peaks."""
    d = {"ms": t_ms, "algorithmic_bytes": alg_bytes,
         "algorithmic_GB/s": alg_bytes / (t_ms / 1e3) / 1e9,
         "algorithmic_over_hbm_peak": alg_bytes / (t_ms / 1e3) / 1e9 / hbm}
    dram = load_traffic(workload, "bag_kernel", "dram") if workload else None
    l2 = load_traffic(workload, "bag_kernel", "l2") if workload else None
    l2_peak = load_l2_peak()
    if dram:
        d.update({"dram_bytes_ncu": dram, "dram_GB/s": dram / (t_ms / 1e3) / 1e9,
                  "frac_hbm_dram": dram / (t_ms / 1e3) / 1e9 / hbm})
    if l2:
        d.update({"l2_bytes_ncu": l2, "l2_GB/s": l2 / (t_ms / 1e3) / 1e9})
        if l2_peak:
            d.update({"l2_peak_GB/s": l2_peak, "frac_l2": l2 / (t_ms / 1e3) / 1e9 / l2_peak})
    return d


def train_timing(steps=8, warmup=2):
    """The data-parallel training step of SURVEY 8f rank 4 at the mid config on one GPU: forward +
    window-routed BCE (2 objectives x 3 Zipper windows = the 6 heads) + backward of the towers and
    the last block's MLP + SGD (TowerTrainer(train_mlp=True)), eager launches, device time per
    step. Not the headline: the reference defines no training step."""
    import torch
    import paper_2512_09200_b200 as L
    from paper_2512_09200_b200.train import TowerTrainer
    c, B = MID, MID_B
    n, d = c["n"], c["d"]
    net = L.Network(**c, max_batch=B, weight_seed=SEED_W)
    tab = torch.empty((n, MID_ROWS, d), dtype=torch.bfloat16, device="cuda")
    L.fill_tables(tab, SEED_T)
    ptrs = torch.tensor([t.data_ptr() for t in tab.unbind(0)], dtype=torch.int64, device="cuda")
    rows = torch.full((n,), MID_ROWS, dtype=torch.int64, device="cuda")
    offsets, ids = L.synth_bags(n, B, MID_MAXLEN, MID_ROWS, SEED_D)
    dom = L.synth_domains(B, c["domains"], SEED_D)
    imp = L.synth_impressions(B, 2, 7)
    win, lab, _ = L.zipper_assign_labels(*imp, [5400000, 86400000, 604800000], [1 / 3] * 3, 7)
    tr = TowerTrainer(net, lr=0.05, train_mlp=True)
    logits = torch.empty((B, c["heads"]), dtype=torch.float32, device="cuda")
    losses = []

    def step():
        net.forward(dom, offsets, ids, ptrs, rows, torch.bfloat16, logits=logits)
        return tr.step(logits, win, lab, 2, 3)

    for _ in range(warmup):
        losses.append(float(step()))
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        loss = step()
    e1.record()
    torch.cuda.synchronize()
    losses.append(float(loss))
    ms = e0.elapsed_time(e1) / steps
    return {"metric": "training samples/s (forward + routed BCE + backward of towers and last-block MLP + SGD)",
            "value": B / (ms / 1e3), "unit": "samples/s", "ms_per_step": ms, "steps": steps,
            "trained_parameters": int(tr.bucket.numel() - 1), "loss_first_last": [losses[0], losses[-1]],
            "launch": "eager (the tower backward reads its domain segment sizes once per step)"}


def zipper_timing(steps=20):
    """K5 Zipper (window assignment + labels, full-portfolio shape: 4 tasks x 3 windows) on
    65,536 impressions per step on the GPU, beside the reference's own zip_dataset
    (datasets.hpp:199-249 compiled in place, oracle/_ref) on one host core."""
    import numpy as np
    import torch
    import oracle
    import paper_2512_09200_b200 as L
    n, T = 65536, FULL_TASKS
    probs = [1.0 / len(FULL_WINDOWS)] * len(FULL_WINDOWS)
    imp = L.synth_impressions(n, T, 7)
    for _ in range(3):
        L.zipper_assign_labels(*imp, FULL_WINDOWS, probs, 7, check_errors=False)
    torch.cuda.synchronize()
    # replayed from a graph: the kernel's device time, not the host's ctypes/allocation overhead
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(steps):
            L.zipper_assign_labels(*imp, FULL_WINDOWS, probs, 7, check_errors=False)
    g.replay()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    g.replay()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    out = {"impressions_per_step": n, "tasks": T, "windows": len(FULL_WINDOWS), "gpu_ms": ms,
           "gpu_impressions_per_s": n / (ms / 1e3)}
    if oracle.ref_available():
        users, ads, ts, conv, pres = oracle.synth_impressions(8192, T, 7)
        t0 = time.perf_counter()
        k = 0
        while time.perf_counter() - t0 < 3.0 or k == 0:
            rc, _, _, _ = oracle.ref_zip_dataset(users, ads, ts, conv, pres, FULL_WINDOWS, probs, 7)
            assert rc == 0
            k += 1
        dt = time.perf_counter() - t0
        out.update({"reference_cpu_impressions_per_s": k * 8192 / dt, "reference_cores": 1,
                    "reference_sample": f"{k} x 8192 impressions through lattice::zip_dataset (oracle/_ref, "
                                        f"records built from columns inside the timed call)"})
    return out


def cpu_baseline_mid(seconds=15.0, threads=None, large=False):
    """Oracle port of the mid (or large) forward (embedding bag + network, fp64) on a bounded sample."""
    import numpy as np
    import oracle
    c = LARGE if large else MID
    table_rows = LARGE_ROWS if large else MID_ROWS
    threads = threads or os.cpu_count() or 1
    lib = oracle.load_oracle()
    n, d = c["n"], c["d"]
    # weights from the counter-based generator, on the host (no GPU needed for this leg)
    w = host_weights(c)
    o, i = oracle.synth_bags(n, 512, MID_MAXLEN, table_rows, SEED_D)
    dom = oracle.synth_domains(512, c["domains"], SEED_D)
    cfg, ws, keep = oracle_net(c, w)
    t0 = time.perf_counter()
    done = 0
    chunk = max(threads, 4)
    while time.perf_counter() - t0 < seconds and done + chunk <= 512:
        pooled, _ = oracle.embedding_bag_synth(SEED_T, n, table_rows, d, 512, o, i, done, done + chunk, threads)
        out = np.zeros((chunk, c["heads"]), np.float32)
        dd = np.ascontiguousarray(dom[done:done + chunk])
        lib.lo_net_forward(oracle.ctypes.byref(cfg), oracle.ctypes.byref(ws), chunk, oracle.ptr(pooled),
                           oracle.ptr(dd), oracle.ptr(out), threads)
        done += chunk
    dt = time.perf_counter() - t0
    return {"value": done / dt, "unit": "samples/s", "cores": threads, "kind": "port",
            "sample": f"{done} samples of the {'large' if large else 'mid'} batch ({dt:.1f} s; tables "
                      f"regenerated lazily; rate extrapolated to the full batch)"}


_HOST_W = {}


def host_weights(c):
    """Mid weights via the oracle generator (bf16-exact), cached."""
    import numpy as np
    import oracle
    key = json.dumps(c, sort_keys=True)
    if key in _HOST_W:
        return _HOST_W[key]
    lib = oracle.load_oracle()

    def tensor(block, kind, index, out_f, fan_in):
        buf = np.zeros((out_f, fan_in), np.float32)
        lib.lo_fill_weights(oracle.ptr(buf), out_f, fan_in, SEED_W, lib.lo_weight_tag(block, kind, index))
        return buf

    w = {"YT": [], "WL": [], "mlp": []}
    for blk in range(c["blocks"]):
        w["YT"].append(tensor(blk, 1, 0, c["k"], c["n"]))
        w["WL"].append(tensor(blk, 2, 0, c["nL"], c["n"]))
        for li in range(len(c["mlp"]) - 1):
            w["mlp"].append(tensor(blk, 3, li, c["mlp"][li + 1], c["mlp"][li]))
    nd = c["n"] * c["d"]
    w["T1"] = np.stack([tensor(g, 4, 0, c["tower_hidden"], nd) for g in range(c["domains"])])
    w["T2"] = np.stack([tensor(g, 5, 0, c["heads"], c["tower_hidden"]) for g in range(c["domains"])])
    _HOST_W[key] = w
    return w


def oracle_net(c, w):
    import numpy as np
    import oracle
    cfg = oracle.LoNetCfg()
    cfg.n, cfg.d, cfg.blocks, cfg.nF, cfg.nL, cfg.k = c["n"], c["d"], c["blocks"], c["nF"], c["nL"], c["k"]
    cfg.n_mlp = len(c["mlp"]) - 1
    for i, v in enumerate(c["mlp"]):
        cfg.mlp[i] = v
    cfg.G, cfg.heads, cfg.tower_hidden, cfg.hard, cfg.bf16 = c["domains"], c["heads"], c["tower_hidden"], 0, 1
    keep = [np.ascontiguousarray(a, dtype=np.float32) for a in w["YT"] + w["WL"] + w["mlp"]]
    nb = c["blocks"]
    P = oracle.ctypes.c_void_p
    yt = (P * nb)(*[a.ctypes.data for a in keep[:nb]])
    wl = (P * nb)(*[a.ctypes.data for a in keep[nb:2 * nb]])
    ml = (P * len(w["mlp"]))(*[a.ctypes.data for a in keep[2 * nb:]])
    T1 = np.ascontiguousarray(w["T1"], dtype=np.float32)
    T2 = np.ascontiguousarray(w["T2"], dtype=np.float32)
    keep += [T1, T2, yt, wl, ml]
    ws = oracle.LoNetWeights(oracle.ctypes.cast(yt, P), oracle.ctypes.cast(wl, P), oracle.ctypes.cast(ml, P),
                             P(T1.ctypes.data), P(T2.ctypes.data))
    return cfg, ws, keep


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--workload", default="mid", choices=["mid", "full", "large", "micro"])
    ap.add_argument("--dtype", default="f32", choices=["f32", "bf16"], help="micro table dtype")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    ap.add_argument("--no-graph", dest="graph", action="store_false",
                    help="launch every kernel of the timed steps from the host instead of replaying the "
                         "forward step from a CUDA graph")
    ap.add_argument("--no-micro", dest="micro", action="store_false",
                    help="mid at N=1: skip the configs[1] micro lines and the Zipper timing")
    ap.add_argument("--exchange", default="peer", choices=["peer", "nccl", "peer1"],
                    help="N>1 sharded embedding exchange: peer memory (default) or NCCL all-to-alls")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    if args.impl == "reference":
        rank = int(os.environ.get("RANK", "0"))
        if rank != 0:
            return
        per_step = max(0.5, min(3.0, 60.0 / (args.warmup + args.steps)))
        if args.workload == "large":
            base = lambda seconds: cpu_baseline_mid(seconds, large=True)
        elif args.workload in ("mid", "full"):
            base = cpu_baseline_mid
        else:
            base = cpu_baseline_micro
        steps = [base(seconds=per_step) for _ in range(args.warmup + args.steps)]
        v = statistics.median([s["value"] for s in steps[args.warmup:]])
        cb = dict(steps[-1])
        cb["value"] = v
        if args.workload == "large":
            metric = "Lattice Network samples/sec (large config, forward step)"
            wl = ("large Lattice Network (CPU oracle port, fp64 with bf16 rounding emulation): 512 tables x "
                  "1.5M rows x 128, l=4, n=512, MLP 16384-2048-2048-32768, B=65536/GPU")
            dtype = "f64"
        elif args.workload in ("mid", "full"):
            metric = "Lattice Network samples/sec (mid config, forward step)"
            wl = ("mid Lattice Network (CPU oracle port, fp64 with bf16 rounding emulation): "
                  "256 sparse feats x 100k rows x 128, l=4, B=32768")
            dtype = "f64"
        else:
            metric = "embedding-bag samples/sec (configs[1] microbench)"
            wl = "micro: 64 tables x 1M rows x 128, B=16384, bags U[0,40]"
            dtype = "f32"
        print(json.dumps({"impl": "reference", "metric": metric, "value": v, "unit": "samples/s",
                          "n_gpus": 0, "steps": args.steps, "warmup": args.warmup,
                          "higher_is_better": True, "config": {"workload": wl}, "dtype": dtype,
                          "data": "synthetic", "cpu_baseline": cb,
                          "e2e": {"value": v, "unit": "samples/s", "h2d_bytes_per_step": 0,
                                  "d2h_bytes_per_step": 0}}))
        return

    rank, world, local = dist_setup(args.gpus)
    if args.workload in ("mid", "full", "large"):
        res = run_mid(args, rank, world, local)
        base = cpu_baseline_mid
    else:
        res, _ = run_micro(args, rank, world, local)
        base = cpu_baseline_micro
    if world == 1 and args.workload == "mid" and args.micro:
        # configs[1] beside the headline: the embedding-bag microbench in both table dtypes, where
        # HBM (not L2) is the bound, each with its own clock samples
        import torch
        torch.cuda.empty_cache()
        res["micro"] = {}
        for dt in ("bf16", "f32"):
            m, _ = run_micro(args, rank, world, local, dtype=dt, min_seconds=1.5)
            m["roofline"]["dram_bytes_ncu"] = load_traffic(f"micro_{dt}", "bag_kernel", "dram")
            if m["roofline"]["dram_bytes_ncu"]:
                m["roofline"]["frac_hbm_dram"] = (m["roofline"]["dram_bytes_ncu"] / (m["roofline"]["kernel_ms_mean"] / 1e3)
                                                  / 1e9 / m["roofline"]["peak"])
            res["micro"][dt] = {k: m[k] for k in ("metric", "value", "unit", "steps", "ms_per_step", "dtype", "roofline",
                                                  "e2e", "clocks")}
            torch.cuda.empty_cache()
        res["zipper"] = zipper_timing()
        torch.cuda.empty_cache()
        try:
            res["train"] = train_timing()
        except Exception as e:  # informational sub-object: never fail the headline line
            res["train"] = {"error": f"{type(e).__name__}: {e}"[:300]}
        torch.cuda.empty_cache()
    if rank == 0:
        if world == 1 and args.workload != "large":
            res["cpu_baseline"] = base(args.cpu_seconds)
            one = base(max(3.0, args.cpu_seconds / 2), threads=1)
            res["cpu_baseline"]["threads_1"] = {k: one[k] for k in ("value", "unit", "cores", "sample")}
        print(json.dumps(res))
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
