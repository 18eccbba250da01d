mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_fullsize.py -q -W error::DeprecationWarning 2>&1 | tail -2
timeout 900 python bench.py > gpurun_out/bench_check.log 2>&1; echo bench=$?
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref_check.log 2>&1; echo bench_ref=$?
python - <<'PY'
import json
for f in ('gpurun_out/bench_check.log','gpurun_out/bench_ref_check.log'):
    for l in open(f):
        if l.startswith('{'):
            d=json.loads(l); print(f, d['value'], d.get('cpu_baseline',{}).get('value'), d.get('e2e',{}).get('value'), (d.get('parity') or {}).get('pass'))
PY
ls /dev/shm | wc -l
