#!/bin/bash
# round-end measurement on one box: GPU tests, smoke, bench lines of every config
mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q > gpurun_out/gputests.log 2>&1; echo "pytest rc $?"; tail -n 3 gpurun_out/gputests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc $?"; tail -n 2 gpurun_out/smoke.log
for c in 4 0 1 2 3 3b; do
  python bench.py --config $c > gpurun_out/b$c.json 2> gpurun_out/b$c.err; echo "bench $c rc $?"
  python - <<P
import json
try:
    d=json.loads(open('gpurun_out/b$c.json').read().strip().splitlines()[-1])
    print('cfg$c %.4e  %.3f ms  e2e %.4e  frac %.3f launches %d  clocks %s' % (d['value'], d['ms_per_step'], d['e2e']['value'], d['roofline']['frac'], d['gpu_launches'], d['clocks']))
except Exception as e: print('cfg$c parse failed', e)
P
done
python bench.py --impl reference > gpurun_out/bref.json 2> gpurun_out/bref.err; echo "ref rc $?"; tail -c 600 gpurun_out/bref.json
