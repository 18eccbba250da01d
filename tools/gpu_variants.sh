mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?; tail -2 gpurun_out/pytest_gpu.log
for rep in 1 2; do
for v in base staged; do
  for c in C4 C3; do
    FEK_LIB_OVERRIDE=tools/exp/libfek_$v.so timeout 300 python tools/profile_case.py --case $c --launches 5 2>&1 | sed "s/^/$v /" | tail -1
  done
  FEK_LIB_OVERRIDE=tools/exp/libfek_$v.so timeout 300 python tools/profile_case.py --case C4 --dtype f32 --launches 5 2>&1 | sed "s/^/$v /" | tail -1
done
done
