mkdir -p gpurun_out/r02c
for rep in 1 2; do for lib in base cur; do
  [ $lib = base ] && L=paper_2504_02211_b200/libefta_b200_base.so || L=paper_2504_02211_b200/libefta_b200.so
  for m in efta-opt none; do
  echo -n "$lib " ; EFTA_LIB=$L timeout 120 python tools/prof_attn.py --mode $m --b 4 --h 32 --s 8192 --d 128 --iters 2 --time --causal
  echo -n "$lib " ; EFTA_LIB=$L timeout 120 python tools/prof_attn.py --mode $m --b 16 --h 16 --s 2048 --d 64 --iters 2 --time --causal
  done
done; done 2>&1 | tee gpurun_out/r02c/ab.log
