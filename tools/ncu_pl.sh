#!/bin/bash
# ncu evidence for the power-law config (BASELINE configs[3]): launch lists and
# full captures of the two-kernel engine and fused variant D.
OUT=gpurun_out; mkdir -p $OUT
make -s -C paper_2105_06176_b200/csrc >/dev/null 2>&1
for eng in two fused-d; do
  common="python bench.py --config powerlaw-22 --engine $eng --no-north-star --no-e2e --no-cpu --no-tts"
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv \
     --log-file $OUT/launches_pl_${eng}.csv $common --steps 20 --warmup 3 > $OUT/ncu_launch_pl_${eng}.json 2>&1
  echo "launches $eng rc=$?"
done
timeout 900 ncu --set full --clock-control none --import-source on -k 'regex:gated_spmv|pipecg_k1' -s 6 -c 3 \
   -o $OUT/prof_pl_two -f python bench.py --config powerlaw-22 --engine two --no-north-star --no-e2e --no-cpu --no-tts --steps 6 --warmup 3 > $OUT/ncu_full_pl_two.log 2>&1
echo "full two rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k 'regex:fused_kernel_d' -s 4 -c 1 \
   -o $OUT/prof_pl_d -f python bench.py --config powerlaw-22 --engine fused-d --no-north-star --no-e2e --no-cpu --no-tts --steps 6 --warmup 3 > $OUT/ncu_full_pl_d.log 2>&1
echo "full d rc=$?"
