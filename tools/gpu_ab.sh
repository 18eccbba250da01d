# same-session A/B of experiment builds: bash tools/gpu_ab.sh "CASES" "VARIANTS" [reps] [extra profile_case args]
mkdir -p gpurun_out
for rep in $(seq 1 ${3:-2}); do for c in $1; do for v in $2; do
  FEK_LIB_OVERRIDE=tools/exp/libfek_$v.so timeout 300 python tools/profile_case.py --case $c --launches 8 $4 2>&1 | sed "s/^/$v /" | tail -1
done; done; done
