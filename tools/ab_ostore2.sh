mkdir -p gpurun_out/r02o
for rep in 1 2; do for lib in base cur; do
  [ $lib = base ] && L=paper_2504_02211_b200/libefta_b200_base.so || L=paper_2504_02211_b200/libefta_b200.so
  for t in "" "--tok"; do
    echo -n "$lib " ; EFTA_LIB=$L timeout 120 python tools/prof_attn.py --mode efta-opt --b 2 --h 20 --s 8192 --d 64 --iters 2 --time $t
    echo -n "$lib " ; EFTA_LIB=$L timeout 120 python tools/prof_attn.py --mode efta-opt --b 1 --h 20 --s 16384 --d 64 --iters 2 --time $t
    echo -n "$lib " ; EFTA_LIB=$L timeout 120 python tools/prof_attn.py --mode none --b 1 --h 20 --s 16384 --d 64 --iters 2 --time $t
  done
done; done 2>&1 | tee gpurun_out/r02o/ab2.log
