# round-1 final: tests, smoke, bench (both arms), ncu captures of the final kernels, launch list
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -2 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
timeout 900 python bench.py > gpurun_out/bench_final.log 2>&1; echo bench=$?
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref_final.log 2>&1; echo bench_ref=$?
for c in C2 C4 C1 C3; do
  python tools/profile_case.py --case $c --launches 4 > gpurun_out/plain_$c.log 2>&1 && \
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:integrate_kernel -s 2 -c 1 -o gpurun_out/prof_${c}_r01 -f python tools/profile_case.py --case $c --launches 4 > gpurun_out/ncu_$c.log 2>&1; echo ncu_$c=$?
done
python tools/profile_case.py --case C4 --dtype f32 --launches 4 > gpurun_out/plain_C4f32.log 2>&1 && \
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:integrate_kernel -s 2 -c 1 -o gpurun_out/prof_C4f32_r01 -f python tools/profile_case.py --case C4 --dtype f32 --launches 4 > gpurun_out/ncu_C4f32.log 2>&1; echo ncu_C4f32=$?
python bench.py --steps 5 --warmup 3 --no-cases --no-cpu --no-e2e > gpurun_out/bench_small.log 2>&1 && \
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r01.csv python bench.py --steps 5 --warmup 3 --no-cases --no-cpu --no-e2e > gpurun_out/ncu_launches.log 2>&1; echo launches=$?
cat gpurun_out/plain_*.log | cut -c1-160
