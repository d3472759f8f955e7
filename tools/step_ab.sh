#!/bin/bash
# whole-step A/B of env knobs at C3 (bench.py --no-nested, alternating runs)
# usage (under gpurun): tools/step_ab.sh "NAME=ENV ..." ...
run() { env $2 python bench.py --steps 20 --warmup 5 --no-nested --cpu-sample-s 0.5 ${BENCH_ARGS} 2>/dev/null | tail -n 1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1', round(d['value']), round(d['ms_per_step'], 3), d['clocks']['sm_mhz'])"; }
for rep in $(seq 1 ${REPS:-2}); do
  for spec in "$@"; do run "${spec%%:*}" "${spec#*:}"; done
done
