#!/bin/bash
# mid bench with the persisting-L2 carve-out set (cudaLimitPersistingL2CacheSize) to 0 / 32 / 64 /
# 96 MB before the run: can evict_last table rows survive the dense part between two steps?
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
for MB in 0 32 64 96 0; do
  python - $MB <<'PY' >> gpurun_out/r40_l2persist.log 2>&1
import ctypes, json, subprocess, sys
mb = int(sys.argv[1])
import torch
torch.cuda.init()
rt = ctypes.CDLL("/usr/local/cuda/lib64/libcudart.so.12")
torch.zeros(1, device="cuda")
rc = rt.cudaDeviceSetLimit(0x06, ctypes.c_size_t(mb << 20))
val = ctypes.c_size_t(0)
rt.cudaDeviceGetLimit(ctypes.byref(val), 0x06)
sys.argv = ["bench.py", "--no-micro", "--cpu-seconds", "1", "--steps", "30"]
import runpy, io, contextlib
buf = io.StringIO()
with contextlib.redirect_stdout(buf):
    runpy.run_path("bench.py", run_name="__main__")
d = json.loads(buf.getvalue().strip().splitlines()[-1])
print(json.dumps({"persist_MB": mb, "rc": rc, "limit": val.value, "value": d["value"], "ms": d["ms_per_step"],
                  "bag_ms": d["stages"]["embedding"]["ms"], "clocks": d["clocks"]["sm_mhz"]}))
PY
done
