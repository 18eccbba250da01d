mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -x -q -s -k "prism or C4 or C3 or every or twisted or unit or identical or errors" > gpurun_out/pytest_refk.log 2>&1; echo pytest=$?
grep -E "max rel err|passed|failed" gpurun_out/pytest_refk.log | tail -5
for rep in 1 2; do for v in base refk; do
  FEK_LIB_OVERRIDE=tools/exp/libfek_$v.so timeout 300 python tools/profile_case.py --case C4 --launches 8 2>&1 | sed "s/^/$v /" | tail -1
done; done
