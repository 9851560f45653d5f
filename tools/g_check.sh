#!/bin/bash
# engine 3 (fused-g) check: irregular parity tests, then power-law 2^22 timings
# per engine, kernel instance and L2 policy (one box, so the A/B is same-box).
#   G_TESTS=0 to skip the tests; G_CFGS="tag:VAR=v,VAR=v tag2:..." variants
set -u
OUT=gpurun_out; mkdir -p $OUT
if [ "${G_TESTS:-1}" = 1 ]; then
timeout 900 python -m pytest tests/test_gpu_irregular.py tests/test_gpu_config_scale.py tests/test_gpu_edge.py -q -m gpu -k "irregular or powerlaw or fused_g or sell or hub or edge" > $OUT/g_tests.txt 2>&1
echo "tests rc=$?" >> $OUT/g_tests.txt; tail -5 $OUT/g_tests.txt
fi
B="python bench.py --config ${G_CONFIG:-powerlaw-22} --no-north-star --no-e2e --no-cpu --no-tts --no-pcg --steps 200 --warmup 10"
one() {  # tag engine env-list
  local tag=$1 eng=$2 envs=$3
  env $(echo "$envs" | tr ',' ' ') timeout 300 $B --engine $eng > $OUT/g_bench_$tag.json 2>/dev/null
  python -c "import json; d=json.loads(open('$OUT/g_bench_$tag.json').read().strip().splitlines()[-1]); print('$tag', round(d['value'],1), 'it/s', round(d['ms_per_step']*1e3,1),'us frac', round(d['roofline']['frac'],3))" 2>&1 | tail -1
}
one two two X=1
for c in ${G_TWO_CFGS:-}; do
  one ${c%%:*} two ${c#*:}
done
for c in ${G_CFGS:-"def:X=1"}; do
  one ${c%%:*} fused-g ${c#*:}
done
