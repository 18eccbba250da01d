# variant x layout x lane-width sweep of the current kernels into the reference's CSV schema
mkdir -p gpurun_out
for c in C1 C2 C3 C4; do
  timeout 900 python -m paper_1504_01023_b200.tune --case $c --elements 2000000 --out gpurun_out/tune_r01_$c.csv > /dev/null 2> gpurun_out/tune_$c.log; echo tune_$c=$?; tail -1 gpurun_out/tune_$c.log
done
