#!/bin/bash
# One gpurun call: any of  tests[=<pytest args>]  bench[=<bench args>]  ncu[=<config>:<engine>]
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
      tag=$(echo "$args" | tr -c 'a-zA-Z0-9-' '_' | cut -c1-40)
      timeout 900 python bench.py $args > $OUT/bench$tag.json 2> $OUT/bench$tag.err; echo "bench $args rc=$?"
      tail -c 4000 $OUT/bench$tag.json; tail -5 $OUT/bench$tag.err ;;
    ncu*)
      spec="${job#ncu}"; spec="${spec#=}"; cfg="${spec%%:*}"; eng="${spec##*:}"
      cfg=${cfg:-3d7-256}; [ "$eng" = "$spec" ] && eng=fused-c; eng=${eng:-fused-c}
      case "$eng" in fused-c) kre='regex:pipecg_fused_kernel_a';; fused-a) kre='regex:pipecg_fused_kernel_a';;
                     fused-b) kre='regex:pipecg_fused_kernel[^_]';; two) kre='regex:sell_spmv|gated_spmv|pipecg_k1';;
                     fused-e|fused-f) kre='regex:pipecg_fused_kernel_s';;
                     fused-g) kre='regex:pipecg_fused_kernel_g';;
                     *) kre='regex:pipecg_';; esac
      common="python bench.py --config $cfg --engine $eng --no-north-star --no-e2e --no-cpu --no-tts --no-pcg"
      timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv \
         --log-file $OUT/launches_${cfg}_${eng}.csv $common --steps 20 --warmup 3 > $OUT/ncu_launch_${cfg}_${eng}.json 2>&1
      echo "ncu launches $cfg $eng rc=$?"
      timeout 900 ncu --set full --clock-control none --import-source on -k "$kre" -s 4 -c 1 \
         -o $OUT/prof_${cfg}_${eng} -f $common --steps 8 --warmup 3 > $OUT/ncu_full_${cfg}_${eng}.log 2>&1
      echo "ncu full $cfg $eng rc=$?"; tail -2 $OUT/ncu_full_${cfg}_${eng}.log ;;
    *) eval "$job" ;;
  esac
done
