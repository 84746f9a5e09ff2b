#!/bin/bash
python bench.py --config 0 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('cfg0 %.4e  %.3f ms  e2e %.4e  launches %d  clocks %s' % (d['value'], d['ms_per_step'], d['e2e']['value'], d['gpu_launches'], d['clocks']))"
