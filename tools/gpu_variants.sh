for rep in 1 2; do for v in base px2; do
  FEK_LIB_OVERRIDE=tools/exp/libfek_$v.so timeout 300 python tools/profile_case.py --case C3 --dtype f32 --launches 8 2>&1 | sed "s/^/$v /" | tail -1
done; done
FEK_LIB_OVERRIDE=tools/exp/libfek_px2.so timeout 300 python tools/profile_case.py --case C3 --dtype f32 --launches 3 --layout-width 8 2>&1 | sed "s/^/px2 W8 /" | tail -1
FEK_LIB_OVERRIDE=tools/exp/libfek_base.so timeout 300 python tools/profile_case.py --case C3 --dtype f32 --launches 3 --layout-width 8 2>&1 | sed "s/^/base W8 /" | tail -1
