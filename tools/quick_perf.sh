#!/bin/bash
# quick kernel-only timings (checksums_ready) at the bench shapes; outputs in gpurun_out/perf.log
mkdir -p gpurun_out
for m in efta-opt none; do
  python tools/prof_attn.py --mode $m --b 32 --h 32 --s 8192 --d 128 --iters 2 --time
  python tools/prof_attn.py --mode $m --b 16 --h 16 --s 2048 --d 64 --iters 2 --time
done 2>&1 | tee -a gpurun_out/perf.log
