#!/bin/bash
# Same-box A/B of library builds (development): tests/dev_abn.sh MODE lib1 lib2 ... ;
# MODE is a tests/dev_ab.py argument list (quoted), "" for its default cases.
# Interleaves the builds over 2 rounds; logs go to gpurun_out/abn_<name>_<round>.log.
mode="$1"; shift
for r in 1 2; do
  for lib in "$@"; do
    n=$(basename "$lib" .so)_$(echo "$mode" | tr -c "a-z0-9\n" "_")
    PBGK_LIB="$lib" python tests/dev_ab.py $mode > "gpurun_out/abn_${n}_$r.log" 2>&1
  done
done
