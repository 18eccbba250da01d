#!/bin/bash
# sass_mix.sh CASE_TU KERNEL_PATTERN "FLAGS" -> register use and instruction mix of one kernel
R=/root/repo; CS=$R/paper_1504_01023_b200/csrc
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++20 --fmad=false -Xcompiler -fPIC -I$R/include -DFEK_QSS_ONLY $3 \
  -Xptxas -v -c $CS/cases/$1.cu -o /tmp/mix_$1.o 2>&1 | grep -A1 "$2" | grep -o "Used [0-9]* registers\|[0-9]* bytes spill stores" | tr '\n' ' '
cuobjdump -sass -fun "$(cuobjdump -symbols /tmp/mix_$1.o | grep -o "_Z[^ ]*$2[^ ]*" | head -1)" /tmp/mix_$1.o > /tmp/mix_$1.sass 2>/dev/null
S=/tmp/mix_$1.sass
echo "FFMA2 $(grep -c 'FFMA2' $S) FMUL2 $(grep -c 'FMUL2' $S) FFMA $(grep -cw 'FFMA' $S) FMUL $(grep -cw 'FMUL' $S) DFMA $(grep -c 'DFMA' $S) MOV $(grep -c ' MOV ' $S) total $(grep -c '/\*[0-9a-f]\{4\}\*/' $S)"
