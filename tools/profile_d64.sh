#!/bin/bash
# d=64 profiling pass (C3 attention shape: B=16 H=16 S=2048 d=64), one GPU, outputs in gpurun_out/.
set -x
mkdir -p gpurun_out
OUT=gpurun_out
python tools/prof_attn.py --mode efta-opt --b 16 --h 16 --s 2048 --d 64 --iters 3 --time > $OUT/d64_time.log 2>&1
python tools/prof_attn.py --mode none --b 16 --h 16 --s 2048 --d 64 --iters 3 --time >> $OUT/d64_time.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:efta_attn_pair_kernel -s 1 -c 1 \
    -o $OUT/attn_c3_opt python tools/prof_attn.py --mode efta-opt --b 16 --h 16 --s 2048 --d 64 --iters 2 > $OUT/ncu_c3_opt.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:efta_attn_pair_kernel -s 1 -c 1 \
    -o $OUT/attn_c3_none python tools/prof_attn.py --mode none --b 16 --h 16 --s 2048 --d 64 --iters 2 > $OUT/ncu_c3_none.log 2>&1
ls -la $OUT
