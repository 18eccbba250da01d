mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_meshgen.py -x -q > gpurun_out/pytest_meshgen.log 2>&1; echo meshgen=$?
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.log 2>&1; echo bench=$?
timeout 600 python bench.py --config C5 --steps 10 --warmup 3 > gpurun_out/bench_c5.log 2>&1; echo bench_c5=$?
tail -3 gpurun_out/pytest_meshgen.log; tail -c 1500 gpurun_out/bench_c5.log
