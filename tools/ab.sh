#!/bin/bash
# same-box A/B of library builds / env switches on one bench config.
#   AB_CONFIG=3d27-400 AB_ENGINE=fused-f AB_RUNS="tag:VAR=v,VAR=v ..." bash tools/ab.sh
set -u
OUT=gpurun_out; mkdir -p $OUT
B="python bench.py --config ${AB_CONFIG:-3d27-400} --engine ${AB_ENGINE:-auto} --no-north-star --no-e2e --no-cpu --no-tts --no-pcg --steps ${AB_STEPS:-60} --warmup 5"
for rep in 1 2; do
for c in ${AB_RUNS}; do
  tag=${c%%:*}; envs=${c#*:}
  env $(echo "$envs" | tr ',' ' ') timeout 600 $B > $OUT/ab_$tag.json 2>$OUT/ab_$tag.err
  python -c "import json; d=json.loads(open('$OUT/ab_$tag.json').read().strip().splitlines()[-1]); print('$tag', round(d['value'],1), 'it/s', round(d['ms_per_step'],4),'ms frac', round(d['roofline']['frac'],3), d['config']['engine'][:8])" 2>&1 | tail -1
done
done
