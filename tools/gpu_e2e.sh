timeout 600 python tools/e2e_diag.py 2>&1 | tail -16
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "host or chunk or ragged" 2>&1 | tail -2
