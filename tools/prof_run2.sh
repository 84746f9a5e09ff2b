#!/bin/bash
# ncu launch lists of the bench commands of configs 2 / 1 (see tools/prof_run.sh)
mkdir -p gpurun_out
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
for c in 2 1; do
  CMD="python bench.py --config $c --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-parareal"
  $CMD > gpurun_out/plain$c.log 2>&1 || { echo "plain $c failed"; continue; }
  ncu --metrics $M --clock-control none -c 700 --csv --log-file gpurun_out/launches_cfg$c.csv $CMD > gpurun_out/ncu_l$c.log 2>&1
  echo "launch list $c rc $?"
done
