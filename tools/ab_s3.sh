# A/B of experiment builds (kernel-only timings, interleaved); VARS="_c1 _c2"
mkdir -p gpurun_out/s3f
L=paper_2504_02211_b200
VARS=${VARS:-"_c1 _c2"}
for v in $VARS; do
  EFTA_LIB=$L/libefta_b200$v.so timeout 300 python -m pytest -x -q tests/test_attention_gpu.py tests/test_fastpath_gpu.py > gpurun_out/s3f/tests$v.log 2>&1
done
for rep in 1 2 3; do
 for v in "" $VARS; do
  for m in efta-opt none; do
   for shp in "--b 16 --h 32 --s 8192 --d 128" "--b 16 --h 16 --s 2048 --d 64"; do
    echo -n "lib$v " >> gpurun_out/s3f/ab_attn.log
    EFTA_LIB=$L/libefta_b200$v.so timeout 100 python tools/prof_attn.py --mode $m $shp --iters 2 --time >> gpurun_out/s3f/ab_attn.log 2>&1
   done
  done
 done
done
