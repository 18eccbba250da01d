for rep in 1 2; do for v in base aeo; do
  for c in C4 C3; do FEK_LIB_OVERRIDE=tools/exp/libfek_$v.so timeout 300 python tools/profile_case.py --case $c --launches 8 2>&1 | sed "s/^/$v /" | tail -1; done
done; done
