#!/bin/bash
python bench.py --config ${1:-2} --steps 3 --warmup 2 --no-cpu-baseline --no-e2e --no-parareal 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['roofline']; print('%s %.4e  %.2f ms  rec share %.3f' % (d['config']['workload'][:5], d['value'], d['ms_per_step'], r.get('recursion_share_of_step') or 0))"
