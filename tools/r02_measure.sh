#!/bin/bash
# Round-2 measurement pass (one gpurun call): bench lines of every config and
# ncu evidence of each config's dominant kernel (launch list + --set full of
# two consecutive launches: an even and an odd iteration of the E/F kernels).
#   bash tools/r02_measure.sh [bench] [ncu]
set -u
OUT=gpurun_out; mkdir -p $OUT
what="${*:-bench ncu}"
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.used --format=csv > $OUT/gpu.txt
if [[ $what == *bench* ]]; then
  timeout 900 python bench.py > $OUT/r02_bench_3d7-256.json 2> $OUT/r02_bench_3d7-256.err; echo "bench 3d7-256 rc=$?"
  for cfg in 3d27-400 powerlaw-22 2d5-512; do
    timeout 1200 python bench.py --config $cfg --no-north-star > $OUT/r02_bench_$cfg.json 2> $OUT/r02_bench_$cfg.err
    echo "bench $cfg rc=$?"
  done
fi
if [[ $what == *ncu* ]]; then
  for spec in "3d7-256:auto:pipecg_fused_kernel_s" "3d27-400:fused-f:pipecg_fused_kernel_s" "3d27-400:fused-e:pipecg_fused_kernel_s" "powerlaw-22:auto:sell_spmv|pipecg_k1|gated_spmv" "2d5-512:auto:pipecg_fused_kernel_p" "powerlaw-22:fused-g:pipecg_fused_kernel_g"; do
    cfg=${spec%%:*}; rest=${spec#*:}; eng=${rest%%:*}; kre=${rest#*:}
    common="python bench.py --config $cfg --engine $eng --no-north-star --no-e2e --no-cpu --no-tts --no-pcg"
    timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv \
       --log-file $OUT/r02_launches_${cfg}_${eng}.csv $common --steps 20 --warmup 3 > /dev/null 2>&1
    n=2; [[ $cfg == powerlaw-22 && $eng == auto ]] && n=3
    timeout 900 ncu --set full --clock-control none --import-source on -k "regex:$kre" -s 6 -c $n \
       -o $OUT/r02_prof_${cfg}_${eng} -f $common --steps 8 --warmup 3 > $OUT/r02_ncu_${cfg}_${eng}.json 2>&1
    echo "ncu $cfg $eng rc=$?"
    # summarise on the box (the reports are tens of MB): launch shares,
    # --set full metrics of every captured launch + their average, the
    # top source lines; the engine code keys profiles/traffic.json
    python tools/ncu_summary.py $OUT/r02_launches_${cfg}_${eng}.csv $OUT/r02_prof_${cfg}_${eng}.ncu-rep \
      --title "r02 $cfg engine $eng" --source profiles/r02_${cfg}_${eng}.md > $OUT/r02_${cfg}_${eng}.md 2>&1
    echo -e "\n## Top source lines (warp-stall samples)\n\n\`\`\`" >> $OUT/r02_${cfg}_${eng}.md
    python tools/ncu_lines.py $OUT/r02_prof_${cfg}_${eng}.ncu-rep 20 >> $OUT/r02_${cfg}_${eng}.md 2>&1
    echo '```' >> $OUT/r02_${cfg}_${eng}.md
    [ "${KEEP_REPS:-0}" = 1 ] || rm -f $OUT/r02_prof_${cfg}_${eng}.ncu-rep
  done
fi
