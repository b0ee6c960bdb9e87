#!/bin/bash
# A/B: kernel-only timing of experiment builds on one box, interleaved (gpurun_out/ab.log)
mkdir -p gpurun_out
VARS=${VARS:-"base _r1"}
for rep in 1 2 3; do
for shape in "--b 16 --h 32 --s 8192 --d 128" "--b 16 --h 16 --s 2048 --d 64"; do
for v in $VARS; do
  for m in ${MODES:-efta-opt none}; do
    [ "$v" = base ] && s="" || s="$v"
    echo -n "lib$v " >> gpurun_out/ab.log
    EFTA_LIB=paper_2504_02211_b200/libefta_b200$s.so timeout 100 python tools/prof_attn.py --mode $m $shape --iters 2 --time >> gpurun_out/ab.log 2>&1
  done
done
done
done
