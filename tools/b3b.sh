#!/bin/bash
python bench.py --config 3b --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-parareal 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['roofline']; print('cfg3b %.4e  %.1f ms  rec share %.3f  launches %d' % (d['value'], d['ms_per_step'], r.get('recursion_share_of_step') or 0, d['gpu_launches']))"
