#!/bin/bash
# Same-box A/B on the config 4 / 2 bench (development): env settings per run,
# e.g. PBGK_LIB=<older build .so> or the plan knobs (PBGK_NS, PBGK_FORCE_A).
run() { echo "== $1 $2"; env $1 timeout 300 python bench.py --no-cpu-baseline --no-e2e --steps 3 --warmup 3 --config $2 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]);r=d['roofline']
print('value %.4g ms/step %.1f sweep_share %.4f sweep_ms_per_step %.2f ms_share %.4f' % (d['value'], d['ms_per_step'], r['sweep_share_of_step'], r['sweep_share_of_step']*d['ms_per_step'], r['multistep_share_of_step']))"; }
for cfg in ${CONFIGS:-4}; do
  for v in ${VARIANTS:-X=0}; do run "$v" $cfg; done
done
