#!/bin/bash
# same-box A/B: tools/ab_run.sh "<python cmd>" lib1 lib2 ... (2 interleaved rounds)
cmd="$1"; shift
for r in 1 2; do
  for lib in "$@"; do
    echo "== $lib round $r"
    PBGK_LIB="$PWD/tools/ablib/$lib.so" $cmd 2>&1 | tail -n 2
  done
done
