mkdir -p gpurun_out
for rep in 1 2; do
for v in A_cta_v2 B_pw_v2 C_pw_loop D_cta_loop; do
  for c in C1 C2 C3 C4; do
    FEK_LIB_OVERRIDE=tools/exp/libfek_$v.so timeout 300 python tools/profile_case.py --case $c --launches 6 2>&1 | sed "s/^/$v /" | tail -1
  done
  FEK_LIB_OVERRIDE=tools/exp/libfek_$v.so timeout 300 python tools/profile_case.py --case C4 --dtype f32 --launches 6 2>&1 | sed "s/^/$v /" | tail -1
  FEK_LIB_OVERRIDE=tools/exp/libfek_$v.so timeout 300 python tools/profile_case.py --case C2 --dtype f32 --launches 6 2>&1 | sed "s/^/$v /" | tail -1
done
done
