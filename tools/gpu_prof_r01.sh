mkdir -p gpurun_out
python tools/probe_peaks.py > gpurun_out/probe.log 2>&1; echo probe=$?
for c in C2 C4 C1 C3; do
  python tools/profile_case.py --case $c --launches 4 > gpurun_out/plain_$c.log 2>&1 && \
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:integrate_kernel -s 2 -c 1 -o gpurun_out/prof_${c}_r01 python tools/profile_case.py --case $c --launches 4 > gpurun_out/ncu_$c.log 2>&1; echo ncu_$c=$?
done
python tools/profile_case.py --case C4 --dtype f32 --launches 4 > gpurun_out/plain_C4f32.log 2>&1 && \
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:integrate_kernel -s 2 -c 1 -o gpurun_out/prof_C4f32_r01 python tools/profile_case.py --case C4 --dtype f32 --launches 4 > gpurun_out/ncu_C4f32.log 2>&1; echo ncu_C4f32=$?
python bench.py --steps 5 --warmup 3 --no-cases --no-cpu --no-e2e > gpurun_out/bench_small.log 2>&1 && \
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r01.csv python bench.py --steps 5 --warmup 3 --no-cases --no-cpu --no-e2e > gpurun_out/ncu_launches.log 2>&1; echo launches=$?
cat gpurun_out/probe.log
