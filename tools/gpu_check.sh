#!/bin/bash
# One gpurun call: any of  tests[=<pytest args>]  bench[=<bench args>]  ncu
# Outputs land in gpurun_out/.
set -u
OUT=gpurun_out
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.used --format=csv > $OUT/gpu.txt
make -s -C paper_2105_06176_b200/csrc >/dev/null 2>&1
make -s -C oracle >/dev/null 2>&1
for job in "$@"; do
  case "$job" in
    tests*)
      args="${job#tests}"; args="${args#=}"
      timeout 1200 python -m pytest tests -q -m gpu $args > $OUT/pytest_gpu.txt 2>&1
      echo "pytest rc=$?" >> $OUT/pytest_gpu.txt; tail -15 $OUT/pytest_gpu.txt ;;
    bench*)
      args="${job#bench}"; args="${args#=}"
      timeout 900 python bench.py $args > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?"
      tail -c 4000 $OUT/bench.json; tail -5 $OUT/bench.err ;;
    ncu)
      timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv \
         --log-file $OUT/launches.csv python bench.py --steps 20 --warmup 3 --no-north-star --no-e2e --no-cpu > $OUT/ncu_launch_bench.json 2>&1
      echo "ncu launches rc=$?"
      timeout 900 ncu --set full --clock-control none --import-source on -k regex:pipecg_fused -s 4 -c 1 \
         -o $OUT/prof_fused -f python bench.py --steps 8 --warmup 3 --no-north-star --no-e2e --no-cpu > $OUT/ncu_full.log 2>&1
      echo "ncu full rc=$?"; tail -2 $OUT/ncu_full.log ;;
    *) eval "$job" ;;
  esac
done
