#!/bin/bash
# development: config 3a iteration-1 rate for the library in PBGK_LIB
python bench.py --config 3 --no-cpu-baseline --no-e2e --no-parareal --steps 3 --warmup 2 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('cfg3a %.4e cell-updates/s  %.2f ms/step' % (d['value'], d['ms_per_step']))"
