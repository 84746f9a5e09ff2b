#!/bin/bash
# development: DRAM bytes of the first msweep launches of a config-4 window per library variant
for lib in "$@"; do
  echo "== $lib"
  PBGK_LIB="$PWD/tools/ablib/$lib.so" ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:msweep_kernel -c 8 --csv python tools/ms_time.py 1 2>/dev/null | python -c "
import csv,sys
rows=[r for r in csv.reader(sys.stdin) if len(r)>10]
h=rows[0]; ik=h.index('Kernel Name'); im=h.index('Metric Name'); iv=h.index('Metric Value'); ii=h.index('ID')
d={}
for r in rows[1:]:
    d.setdefault(r[ii],{'k':r[ik][:40]})[r[im]]=r[iv]
for k,v in d.items(): print(k, v)
"
done
