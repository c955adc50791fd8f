"""Feasibility of overlapping the embedding stage of batch i+1 with the dense part of batch i:
times (a) the mid forward alone, (b) the mid bag kernel alone, (c) both issued together on two
streams (the bag into a scratch buffer), each averaged over 10 back-to-back repetitions.
Prints one JSON line."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    import paper_2512_09200_b200 as L
    import bench
    c, B, R, ML = bench.MID, bench.MID_B, bench.MID_ROWS, bench.MID_MAXLEN
    n, d = c["n"], c["d"]
    net = L.Network(**c, max_batch=B, weight_seed=7)
    tab = torch.empty((n, R, d), dtype=torch.bfloat16, device="cuda")
    L.fill_tables(tab, 5)
    ptrs = torch.tensor([t.data_ptr() for t in tab.unbind(0)], dtype=torch.int64, device="cuda")
    rows = torch.full((n,), R, dtype=torch.int64, device="cuda")
    offsets, ids = L.synth_bags(n, B, ML, R, 11)
    offsets2, ids2 = L.synth_bags(n, B, ML, R, 12)
    dom = L.synth_domains(B, c["domains"], 11)
    logits = torch.empty((B, c["heads"]), dtype=torch.float32, device="cuda")
    out = torch.empty((B, n, d), dtype=torch.bfloat16, device="cuda")
    tl = list(tab.unbind(0))
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()

    def fwd(st):
        net.forward(dom, offsets, ids, ptrs, rows, torch.bfloat16, logits=logits, stream=st)

    def bag(st):
        L.embedding_bag(tl, offsets2, ids2, B, out=out, normalize=True, check_errors=False, table_ptrs=ptrs,
                        rows=rows, stream=st)

    def timed(fn, reps=10):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            fn()
        # join both streams into the current one
        for st in (s1, s2):
            ev = torch.cuda.Event()
            ev.record(st)
            torch.cuda.current_stream().wait_event(ev)
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / reps

    def both():
        ev = torch.cuda.Event()
        ev.record()
        s1.wait_event(ev)
        s2.wait_event(ev)
        fwd(s1)
        bag(s2)

    def fwd_only():
        ev = torch.cuda.Event()
        ev.record()
        s1.wait_event(ev)
        fwd(s1)

    def bag_only():
        ev = torch.cuda.Event()
        ev.record()
        s2.wait_event(ev)
        bag(s2)

    res = {"forward_ms": timed(fwd_only), "bag_ms": timed(bag_only), "forward_and_bag_concurrent_ms": timed(both)}
    res["serial_sum_ms"] = res["forward_ms"] + res["bag_ms"]
    print(json.dumps(res))


if __name__ == "__main__":
    main()
