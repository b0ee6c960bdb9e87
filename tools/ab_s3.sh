# A/B of experiment builds against the HEAD build (kernel-only timings, interleaved)
mkdir -p gpurun_out/s3b
L=paper_2504_02211_b200
EFTA_LIB=$L/libefta_b200_g3.so timeout 300 python -m pytest -x -q tests/test_abft_gemm_gpu.py tests/test_layouts_gpu.py tests/test_attention_gpu.py > gpurun_out/s3b/g3_tests.log 2>&1
for rep in 1 2 3; do
 for v in _head _g3; do
  for shp in "--m 32768 --n 4096 --k 1024" "--m 32768 --n 1024 --k 4096" "--m 16384 --n 5120 --k 1280" "--m 16384 --n 1280 --k 5120"; do
   echo -n "lib$v $shp " >> gpurun_out/s3b/ab_gemm.log
   EFTA_LIB=$L/libefta_b200$v.so timeout 100 python tools/prof_gemm.py $shp >> gpurun_out/s3b/ab_gemm.log 2>&1
  done
  for shp in "--b 16 --h 32 --s 8192 --d 128" "--b 16 --h 16 --s 2048 --d 64" "--b 32 --h 20 --s 512 --d 64"; do
   echo -n "lib$v " >> gpurun_out/s3b/ab_attn.log
   EFTA_LIB=$L/libefta_b200$v.so timeout 100 python tools/prof_attn.py --mode efta-opt $shp --iters 2 --time >> gpurun_out/s3b/ab_attn.log 2>&1
  done
 done
done
