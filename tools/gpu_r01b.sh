mkdir -p gpurun_out
python tools/e2e_diag.py > gpurun_out/e2e_diag.log 2>&1; echo e2e=$?
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
for c in C4 C3; do python tools/profile_case.py --case $c --launches 6 > gpurun_out/plain_$c.log 2>&1 || echo plain_$c failed; done
tail -3 gpurun_out/pytest_gpu.log; cat gpurun_out/plain_*.log gpurun_out/e2e_diag.log
