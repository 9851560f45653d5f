#!/bin/bash
# ncu --set full of one kernel of one engine:  ncu_one.sh <config> <engine> <kernel-regex> <tag> [ENV=V ...]
OUT=gpurun_out; mkdir -p $OUT
cfg=$1; eng=$2; kre=$3; tag=$4; shift 4
make -s -C paper_2105_06176_b200/csrc >/dev/null 2>&1
env "$@" timeout 900 ncu --set full --clock-control none --import-source on -k "regex:$kre" -s 5 -c 1 \
   -o $OUT/prof_$tag -f python bench.py --config $cfg --engine $eng --no-north-star --no-e2e --no-cpu --no-tts --no-pcg --steps 8 --warmup 3 > $OUT/ncu_full_$tag.log 2>&1
echo "ncu $tag rc=$?"; tail -1 $OUT/ncu_full_$tag.log
