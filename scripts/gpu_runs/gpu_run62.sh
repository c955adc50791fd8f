# re-entry check after container restore: full gpu suite, smoke, default bench, reference arm
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?; tail -5 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1; echo smoke rc=$?; tail -2 gpurun_out/smoke.log
timeout 400 python bench.py > gpurun_out/n1.json 2>gpurun_out/n1.err; echo bench rc=$?; tail -1 gpurun_out/n1.json
timeout 400 python bench.py --impl reference > gpurun_out/ref.json 2>gpurun_out/ref.err; echo ref rc=$?; tail -1 gpurun_out/ref.json
