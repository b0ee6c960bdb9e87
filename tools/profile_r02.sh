#!/bin/bash
# Round-2 profiling pass (one GPU, under gpurun). The .ncu-rep files are summarised ON the box
# (tools/ncu_summary.py + raw/source CSV pages) and then deleted so gpurun_out/ stays < 64 MiB.
# usage: bash tools/profile_r02.sh [tag] [which...]   which: c4opt c4none c3opt c3none gemm launches
set -x
TAG=${1:-r02}; shift
WHICH=${@:-"c3opt c3none c4opt c4none gemm launches"}
OUT=gpurun_out/$TAG
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $OUT/gpu.txt
prof() {  # name, kernel regex, command...
  local name=$1 kre=$2; shift 2
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$kre -s 1 -c 1 \
      -o $OUT/$name "$@" > $OUT/ncu_$name.log 2>&1
  python tools/ncu_summary.py $OUT/$name.ncu-rep > $OUT/$name.summary.json
  ncu -i $OUT/$name.ncu-rep --page raw --csv > $OUT/$name.raw.csv 2>/dev/null
  ncu -i $OUT/$name.ncu-rep --page source --csv --print-source sass > $OUT/$name.sass.csv 2>/dev/null
  gzip -f $OUT/$name.sass.csv
  rm -f $OUT/$name.ncu-rep
}
for w in $WHICH; do case $w in
  c3opt) prof c3_opt efta_attn_pair_kernel python tools/prof_attn.py --mode efta-opt --b 16 --h 16 --s 2048 --d 64 --iters 2 ;;
  c3none) prof c3_none efta_attn_pair_kernel python tools/prof_attn.py --mode none --b 16 --h 16 --s 2048 --d 64 --iters 2 ;;
  c4opt) prof c4_opt efta_attn_pair_kernel python tools/prof_attn.py --mode efta-opt --b 32 --h 32 --s 8192 --d 128 --iters 2 ;;
  c4none) prof c4_none efta_attn_pair_kernel python tools/prof_attn.py --mode none --b 32 --h 32 --s 8192 --d 128 --iters 2 ;;
  gemm) prof gemm_c3 abft_gemm_kernel python tools/prof_gemm.py --m 32768 --n 4096 --k 1024 --iters 2 ;;
  launches) timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv \
      python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-campaign --no-suite > $OUT/bench_under_ncu.log 2>&1 ;;
esac; done
python tools/prof_attn.py --mode efta-opt --b 16 --h 16 --s 2048 --d 64 --iters 3 --time > $OUT/time.log 2>&1
python tools/prof_attn.py --mode none --b 16 --h 16 --s 2048 --d 64 --iters 3 --time >> $OUT/time.log 2>&1
du -sh $OUT; ls -la $OUT
