#!/bin/bash
# Round profiling pass (run under gpurun on ONE GPU). Outputs land in gpurun_out/.
set -x
mkdir -p gpurun_out
OUT=gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $OUT/gpu.txt
# 1) launch list of the bench command (cold-cache, serialised: shares, not absolutes)
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv \
    python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-campaign --no-suite > $OUT/bench_under_ncu.log 2>&1
# 2) full sections of the top kernel (protected, bench shape) and its unprotected twin
timeout 900 ncu --set full --clock-control none --import-source on -k regex:efta_attn_pair_kernel -s 1 -c 1 \
    -o $OUT/attn_c4_opt python tools/prof_attn.py --mode efta-opt --b 32 --h 32 --s 8192 --d 128 --iters 2 > $OUT/ncu_opt.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:efta_attn_pair_kernel -s 1 -c 1 \
    -o $OUT/attn_c4_none python tools/prof_attn.py --mode none --b 32 --h 32 --s 8192 --d 128 --iters 2 > $OUT/ncu_none.log 2>&1
# 3) the strided-ABFT FFN GEMM (C3 first FFN GEMM)
timeout 600 ncu --set full --clock-control none --import-source on -k regex:abft_gemm_kernel -s 1 -c 1 \
    -o $OUT/abft_gemm_c3 python tools/prof_gemm.py --m 32768 --n 4096 --k 1024 --iters 2 > $OUT/ncu_gemm.log 2>&1
ls -la $OUT
