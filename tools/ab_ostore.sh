# A/B: current library vs libefta_b200_base.so (HEAD build) on the d=64 shapes and C4, kernel-only
mkdir -p gpurun_out/r02o
for rep in 1 2 3; do for lib in base cur; do
  [ $lib = base ] && L=paper_2504_02211_b200/libefta_b200_base.so || L=paper_2504_02211_b200/libefta_b200.so
  for m in efta-opt none; do
    echo -n "$lib " ; EFTA_LIB=$L timeout 120 python tools/prof_attn.py --mode $m --b 16 --h 16 --s 2048 --d 64 --iters 2 --time
    echo -n "$lib " ; EFTA_LIB=$L timeout 120 python tools/prof_attn.py --mode $m --b 32 --h 20 --s 512 --d 64 --iters 2 --time
  done
done; done 2>&1 | tee gpurun_out/r02o/ab.log
for lib in base cur; do
  [ $lib = base ] && L=paper_2504_02211_b200/libefta_b200_base.so || L=paper_2504_02211_b200/libefta_b200.so
  echo "== $lib"; EFTA_LIB=$L python tools/prof_layer.py --iters 7 2>&1 | grep -o "S=[0-9]* B=[0-9]*: prot/fused [0-9.]* ms\|prot/fused-nogelu [0-9.]* ms [0-9.]* TF/s\|unprot/fused-nogelu [0-9.]* ms [0-9.]* TF/s"
done 2>&1 | tee gpurun_out/r02o/layer.log
