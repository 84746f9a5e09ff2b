#!/bin/bash
# ncu launch lists (time + DRAM bytes per launch) of the bench commands of configs 4 / 3 / 0
# and full captures of the steady msweep / esweep passes; run only after the plain commands exit 0
mkdir -p gpurun_out
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
for c in 4 3 0; do
  CMD="python bench.py --config $c --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-parareal"
  $CMD > gpurun_out/plain$c.log 2>&1 || { echo "plain $c failed"; continue; }
  ncu --metrics $M --clock-control none -c 700 --csv --log-file gpurun_out/launches_cfg$c.csv $CMD > gpurun_out/ncu_l$c.log 2>&1
  echo "launch list $c rc $?"
done
ncu --set full --clock-control none --import-source on -k regex:msweep_kernel -s 6 -c 1 -o gpurun_out/prof_ms_final -f \
  python bench.py --config 4 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-parareal > gpurun_out/ncu_msf.log 2>&1; echo "ms capture rc $?"
ncu --set full --clock-control none --import-source on -k regex:esweep_kernel -s 12 -c 1 -o gpurun_out/prof_es_final -f \
  python bench.py --config 3 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-parareal > gpurun_out/ncu_esf.log 2>&1; echo "es capture rc $?"
