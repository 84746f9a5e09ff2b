#!/bin/bash
python bench.py --config 4 --no-cpu-baseline --no-e2e --no-parareal 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('cfg4 %.4e  %.2f ms  clocks %s' % (d['value'], d['ms_per_step'], d['clocks']))"
