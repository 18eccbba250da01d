#!/bin/bash
# kstat.sh CASE_TU [FLAGS] [PATTERN] -> registers / spills / FP instruction counts of the natural QSS kernel
# (default tile, store mode; no GPU)
PAT=${3:-Li0ELi0EEEEEvNS}
R=/root/repo; CS=$R/paper_1504_01023_b200/csrc
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++20 --fmad=false -Xcompiler -fPIC -I$R/include -DFEK_QSS_ONLY $2 \
  -Xptxas -v -c $CS/cases/$1.cu -o /tmp/ks_$1.o 2>&1 | grep -A3 "Compiling entry.*$PAT" | grep -o "Used [0-9]* registers\|[0-9]* bytes spill stores" | tr '\n' ' '
cuobjdump -sass /tmp/ks_$1.o > /tmp/ks_$1.sass
python3 - /tmp/ks_$1.sass "$PAT" <<'PY'
import re, sys
from collections import Counter
txt = open(sys.argv[1]).read()
for f in re.split(r'\n\s*Function : ', txt)[1:]:
    if sys.argv[2] not in f.split('\n')[0]:
        continue
    ins = re.findall(r'/\*[0-9a-f]{4}\*/\s+(?:@!?U?P\w+\s+)?([A-Z0-9_.]+)', f)
    c = Counter(i.split('.')[0] for i in ins)
    fp64 = sum(c[k] for k in ('DFMA', 'DMUL', 'DADD'))
    fp32 = sum(c[k] for k in ('FFMA', 'FMUL', 'FADD', 'FFMA2', 'FMUL2', 'FADD2'))
    print(f"total {len(ins)} fp64 {fp64} (DFMA {c['DFMA']} DMUL {c['DMUL']} DADD {c['DADD']}) fp32 {fp32}")
PY
