mkdir -p gpurun_out
for rep in 1 2; do for v in base p3; do
  FEK_LIB_OVERRIDE=tools/exp/libfek_$v.so timeout 300 python tools/profile_case.py --case C3 --launches 6 2>&1 | sed "s/^/$v /" | tail -1
done; done
for c in C1 C2 C3 C4; do timeout 900 python -m paper_1504_01023_b200.tune --case $c --elements 2000000 --repeats 5 --out gpurun_out/tune_$c.csv > /dev/null 2> gpurun_out/tune_$c.log; echo tune_$c=$?; tail -1 gpurun_out/tune_$c.log; done
