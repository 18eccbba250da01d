mkdir -p gpurun_out
python tools/profile_case.py --case C4 --launches 4 > gpurun_out/plain.log 2>&1 && \
 timeout 600 ncu --set full --clock-control none --import-source on -k regex:integrate_kernel -s 2 -c 1 -o gpurun_out/prof_C4b python tools/profile_case.py --case C4 --launches 4 > gpurun_out/ncu_C4b.log 2>&1; echo ncu=$?
