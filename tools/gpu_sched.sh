# dynamic tile queue: correctness, then static-vs-dynamic timings and the C5 overlap study
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_scheduler.py -x -q > gpurun_out/pytest_sched.log 2>&1; echo sched_tests=$?
tail -3 gpurun_out/pytest_sched.log
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -3 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
timeout 900 python bench.py --steps 20 --warmup 5 --cases C1,C1static,C3,C3static,C4,C4static,C4f32,C4f32static,C5,C2packed,C2packedstatic > gpurun_out/bench_sched.log 2>&1; echo bench=$?
timeout 600 python tools/c5_overlap.py > gpurun_out/c5_overlap.log 2>&1; echo overlap=$?
tail -30 gpurun_out/c5_overlap.log
