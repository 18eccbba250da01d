mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_invariants.py tests/test_gpu_bounds.py tests/test_gpu_bench_golden.py -x -q -s > gpurun_out/pytest_prism.log 2>&1; echo pytest=$?
grep -E "max rel err|passed|failed|Error" gpurun_out/pytest_prism.log | tail -8
