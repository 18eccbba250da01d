# round-end check, as the driver runs it: GPU tests, smoke(), both bench arms (default flags)
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -2 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref.log 2>&1; echo bench_ref=$?
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo bench=$?
grep -h '^{' gpurun_out/bench.log > gpurun_out/bench_line.json
grep -h '^{' gpurun_out/bench_ref.log > gpurun_out/bench_ref_line.json
# launch list of the bench command (graph-timed steps included), only after it ran clean without ncu
python bench.py --steps 5 --warmup 3 --no-cases --no-cpu --no-e2e > gpurun_out/bench_small.log 2>&1 && \
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${TAG:-r02}.csv \
  python bench.py --steps 5 --warmup 3 --no-cases --no-cpu --no-e2e > gpurun_out/ncu_launches.log 2>&1; echo launches=$?
