# end-of-session state check (1 GPU): full GPU suite, smoke, drop-in, default bench + reference arm
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?; tail -2 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke rc=$?; tail -1 gpurun_out/smoke.log
timeout 300 tests/cpp/test_dropin > gpurun_out/dropin.log 2>&1; echo dropin rc=$?; tail -1 gpurun_out/dropin.log
timeout 400 python bench.py > gpurun_out/n1.json 2>gpurun_out/n1.err; echo bench rc=$?
python -c "
import json
d=json.loads([l for l in open('gpurun_out/n1.json') if l.startswith('{')][-1])
print(round(d['value']), round(d['e2e']['value']), d['ms_per_step'], d['gpu_launches'], round(d['roofline']['frac'],3), d['clocks'])"
timeout 400 python bench.py --impl reference > gpurun_out/ref.json 2>gpurun_out/ref.err; echo ref rc=$?
