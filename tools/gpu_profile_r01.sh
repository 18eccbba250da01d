mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.log 2>&1; echo bench=$?
for c in C2 C4 C1 C3; do python tools/profile_case.py --case $c --launches 4 > gpurun_out/plain_$c.log 2>&1 || echo plain_$c failed; done
python tools/profile_case.py --case C2 --launches 4 > gpurun_out/plain.log 2>&1 && \
 timeout 600 ncu --set full --clock-control none --import-source on -k regex:integrate_kernel -s 2 -c 1 -o gpurun_out/prof_C2 python tools/profile_case.py --case C2 --launches 4 > gpurun_out/ncu_C2.log 2>&1; echo ncuC2=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:integrate_kernel -s 2 -c 1 -o gpurun_out/prof_C4 python tools/profile_case.py --case C4 --launches 4 > gpurun_out/ncu_C4.log 2>&1; echo ncuC4=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:integrate_kernel -s 2 -c 1 -o gpurun_out/prof_C1 python tools/profile_case.py --case C1 --launches 4 > gpurun_out/ncu_C1.log 2>&1; echo ncuC1=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 5 --warmup 3 --no-cases --no-cpu --no-e2e > gpurun_out/ncu_launches.log 2>&1; echo ncu_launches=$?
tail -3 gpurun_out/pytest_gpu.log; cat gpurun_out/plain_*.log
