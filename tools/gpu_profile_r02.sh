# round-2 evidence: launch list of the headline bench command, ncu --set full of each configuration's
# integration kernel (C5 parts first: the headline's kernels), summarised under profiles/
mkdir -p gpurun_out
TAG=${TAG:-r02}
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv \
  python bench.py --steps 5 --warmup 3 --no-cases --no-cpu --no-e2e > gpurun_out/ncu_launches_$TAG.log 2>&1; echo launches=$?
for c in ${CASES:-C5P C5T C1 C2 C3 C4}; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:integrate_kernel -s 2 -c 1 \
    -o gpurun_out/prof_${c}_$TAG -f python tools/profile_case.py --case $c --launches 4 > gpurun_out/ncu_${c}_$TAG.log 2>&1
  echo ncu_$c=$?
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:integrate_kernel -s 2 -c 1 \
  -o gpurun_out/prof_C4f32_$TAG -f python tools/profile_case.py --case C4 --dtype f32 --launches 4 > gpurun_out/ncu_C4f32_$TAG.log 2>&1
echo ncu_C4f32=$?
