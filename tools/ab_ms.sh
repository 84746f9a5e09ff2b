#!/bin/bash
# Development A/B of macro variants of one kernel file (AB_SRC, default msweep):
# tools/ab_ms.sh name "-DX=1 -DY=0" ...
# builds tools/ablib/<name>.so from the working tree with the given nvcc defines
# (only msweep.cu is recompiled; the other objects come from the last full build
# kept in tools/ablib/base/).
set -e
cd "$(dirname "$0")/.."
base=tools/ablib/base
src=${AB_SRC:-msweep}
mkdir -p $base
FL="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xcompiler -O2 -I include"
for f in sweep sweep_a sweep_b sweep_c finalize fluid fsweep msweep esweep marginal capi; do
  [ $f = $src ] && continue
  if [ ! -f $base/$f.o ] || [ paper_2502_02704_b200/csrc/$f.cu -nt $base/$f.o ]; then
    nvcc $FL -c paper_2502_02704_b200/csrc/$f.cu -o $base/$f.o &
  fi
done
wait
while [ $# -gt 0 ]; do
  name=$1; defs=$2; shift 2
  nvcc $FL $defs -Xptxas -v -c paper_2502_02704_b200/csrc/$src.cu -o tools/ablib/ms_$name.o 2> tools/ablib/ms_$name.ptxas.txt
  objs=$(ls $base/*.o | grep -v "/$src.o")
  nvcc -gencode arch=compute_100a,code=sm_100a -shared -o tools/ablib/$name.so $objs tools/ablib/ms_$name.o
  grep -c "spill" tools/ablib/ms_$name.ptxas.txt >/dev/null; echo built $name: $(grep -o "[0-9]* bytes spill stores" tools/ablib/ms_$name.ptxas.txt | sort | uniq -c | tr '\n' ' ')
done
