mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
for c in C1 C2 C3 C4; do timeout 300 python tools/profile_case.py --case $c --launches 6 > gpurun_out/plain_$c.log 2>&1 || echo plain_$c failed; done
timeout 300 python tools/profile_case.py --case C4 --launches 6 --dtype f32 > gpurun_out/plain_C4f32.log 2>&1
tail -3 gpurun_out/pytest_gpu.log; cat gpurun_out/plain_*.log
