for rep in 1 2; do for v in base f32p; do
  FEK_LIB_OVERRIDE=tools/exp/libfek_$v.so timeout 300 python tools/profile_case.py --case C4 --dtype f32 --launches 5 2>&1 | sed "s/^/$v /" | tail -1
  FEK_LIB_OVERRIDE=tools/exp/libfek_$v.so timeout 300 python tools/profile_case.py --case C3 --dtype f32 --launches 5 2>&1 | sed "s/^/$v /" | tail -1
done; done
