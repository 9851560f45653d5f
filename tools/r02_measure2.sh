#!/bin/bash
# Re-measure after a kernel change: bench lines + ncu summaries for given configs.
#   R2_BENCH="3d7-256 3d27-400" R2_NCU="3d7-256:auto:pipecg_fused_kernel_s" bash tools/r02_measure2.sh
set -u
OUT=gpurun_out; mkdir -p $OUT
for cfg in ${R2_BENCH:-}; do
  extra=""; [ "$cfg" != "3d7-256" ] && extra="--no-north-star"
  timeout 1200 python bench.py --config $cfg $extra > $OUT/r02_bench_$cfg.json 2> $OUT/r02_bench_$cfg.err
  echo "bench $cfg rc=$?"
done
for spec in ${R2_NCU:-}; do
  cfg=${spec%%:*}; rest=${spec#*:}; eng=${rest%%:*}; kre=${rest#*:}
  common="python bench.py --config $cfg --engine $eng --no-north-star --no-e2e --no-cpu --no-tts --no-pcg"
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv \
     --log-file $OUT/r02_launches_${cfg}_${eng}.csv $common --steps 20 --warmup 3 > /dev/null 2>&1
  timeout 900 ncu --set full --clock-control none --import-source on -k "regex:$kre" -s 6 -c 2 \
     -o $OUT/r02_prof_${cfg}_${eng} -f $common --steps 8 --warmup 3 > $OUT/r02_ncu_${cfg}_${eng}.json 2>&1
  echo "ncu $cfg $eng rc=$?"
  python tools/ncu_summary.py $OUT/r02_launches_${cfg}_${eng}.csv $OUT/r02_prof_${cfg}_${eng}.ncu-rep \
    --title "r02 $cfg engine $eng" --source profiles/r02_${cfg}_${eng}.md > $OUT/r02_${cfg}_${eng}.md 2>&1
  echo -e "\n## Top source lines (warp-stall samples)\n\n\`\`\`" >> $OUT/r02_${cfg}_${eng}.md
  python tools/ncu_lines.py $OUT/r02_prof_${cfg}_${eng}.ncu-rep 20 >> $OUT/r02_${cfg}_${eng}.md 2>&1
  echo '```' >> $OUT/r02_${cfg}_${eng}.md
  rm -f $OUT/r02_prof_${cfg}_${eng}.ncu-rep
done
