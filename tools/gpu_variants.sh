for rep in 1 2; do for v in base x2; do
  FEK_LIB_OVERRIDE=tools/exp/libfek_$v.so timeout 300 python tools/profile_case.py --case C4 --dtype f32 --launches 8 2>&1 | sed "s/^/$v /" | tail -1
done; done
for v in base x2; do FEK_LIB_OVERRIDE=tools/exp/libfek_$v.so timeout 300 python tools/profile_case.py --case C4 --dtype f32 --launches 3 --layout-width 16 2>&1 | sed "s/^/$v W16 /" | tail -1; done
