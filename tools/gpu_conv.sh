mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_layout_convert.py tests/test_gpu_scheduler.py -x -q > gpurun_out/pytest_conv.log 2>&1; echo tests=$?
tail -3 gpurun_out/pytest_conv.log
timeout 300 python tools/convert_bw.py 2>&1 | tail -6
