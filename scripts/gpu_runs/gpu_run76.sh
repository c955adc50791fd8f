timeout 600 python -m pytest tests/test_network_gpu.py -x -q -k "large_n" > gpurun_out/pytest_large.log 2>&1; echo pytest rc=$?; tail -2 gpurun_out/pytest_large.log
for v in base new base new; do
  if [ $v = base ]; then export LATTICE_LIB=$PWD/ab/base.so; else unset LATTICE_LIB; fi
  echo -n "$v: "; timeout 300 python scripts/fm_large_probe.py 4 2>&1 | tail -1
done | tee gpurun_out/fm_large_ab2.log
