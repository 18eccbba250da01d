mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
timeout 1200 python -m pytest tests -m gpu -x -q -s > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.log 2>&1; echo bench=$?
timeout 600 python bench.py --impl reference --steps 5 --warmup 2 > gpurun_out/bench_ref.log 2>&1; echo bench_ref=$?
grep -E "C[0-9]:|passed|failed" gpurun_out/pytest_gpu.log | tail -6; tail -c 600 gpurun_out/bench_ref.log
