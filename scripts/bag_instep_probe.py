"""Why is the mid bag stage slower inside the step than alone? Times the bag stage (network stage
events) of the mid config (a) in back-to-back eager forwards, (b) after the GPU idled 200 ms
(clocks recover from the GEMMs' power cap), (c) the bag kernel alone back to back
(lattice_embedding_bag, no GEMMs in between). Samples SM clocks with nvidia-smi meanwhile.
Prints one JSON line."""
import json
import os
import statistics
import subprocess
import sys
import time

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
    dom = L.synth_domains(B, c["domains"], 11)
    logits = torch.empty((B, c["heads"]), dtype=torch.float32, device="cuda")
    net.set_timing(True)

    def fwd():
        net.forward(dom, offsets, ids, ptrs, rows, torch.bfloat16, logits=logits)

    for _ in range(3):
        fwd()
    torch.cuda.synchronize()

    def clocks():
        try:
            out = subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm", "--format=csv,noheader,nounits", "-i", "0"],
                                 capture_output=True, text=True, timeout=10).stdout.split()
            return float(out[0])
        except Exception:
            return None

    res = {}
    a = []
    for _ in range(10):
        fwd()
        a.append(net.stage_times()[1])
    res["in_step_back_to_back_ms"] = statistics.median(a)
    res["sm_mhz_after_back_to_back"] = clocks()
    b = []
    for _ in range(6):
        torch.cuda.synchronize()
        time.sleep(0.2)
        fwd()
        b.append(net.stage_times()[1])
    res["after_200ms_idle_ms"] = statistics.median(b)
    net.set_timing(False)
    # the bag kernel alone, back to back, into a scratch pooled buffer
    out = torch.empty((B, n, d), dtype=torch.bfloat16, device="cuda")
    e = [torch.cuda.Event(enable_timing=True) for _ in range(11)]
    tl = list(tab.unbind(0))
    bag = lambda: L.embedding_bag(tl, offsets, ids, B, out=out, normalize=True, check_errors=False,
                                  table_ptrs=ptrs, rows=rows)
    for i in range(3):
        bag()
    torch.cuda.synchronize()
    res["sm_mhz_before_alone"] = clocks()
    for i in range(10):
        e[i].record()
        bag()
    e[10].record()
    torch.cuda.synchronize()
    res["bag_alone_back_to_back_ms"] = statistics.median(e[i].elapsed_time(e[i + 1]) for i in range(10))
    print(json.dumps(res))


if __name__ == "__main__":
    main()
