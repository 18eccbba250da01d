# same-session A/B of experiment builds through bench.py's C5 headline (the driver's regime: 20 steps,
# 5 warm-up, power cap included): bash tools/gpu_bench_ab.sh "VARIANTS" [reps] [extra bench args]
for rep in $(seq 1 ${2:-3}); do for v in $1; do
  FEK_LIB_OVERRIDE=tools/exp/libfek_$v.so timeout 300 python bench.py --no-cases --no-cpu --no-e2e $3 2>/dev/null | grep '^{' | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']['step']['per_kernel_ms']; print('$v', '%.3f' % d['ms_per_step'], d['clocks']['sm_mhz'], {k: round(x, 3) for k, x in r.items()})"
done; done
