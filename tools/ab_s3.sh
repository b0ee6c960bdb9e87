# A/B of an experiment build against the current build (kernel-only timings, interleaved)
mkdir -p gpurun_out/s3n
L=paper_2504_02211_b200
V=${V:-_x1}
EFTA_LIB=$L/libefta_b200$V.so timeout 600 python -m pytest -x -q tests/test_abft_gemm_gpu.py tests/test_layouts_gpu.py tests/test_layer_gpu.py tests/test_cpp_dropin.py > gpurun_out/s3n/tests$V.log 2>&1
for rep in 1 2 3 4; do
 for v in "" $V; do
  for shp in "--m 32768 --n 4096 --k 1024" "--m 32768 --n 1024 --k 4096" "--m 16384 --n 5120 --k 1280" "--m 16384 --n 1280 --k 5120"; do
   echo -n "lib$v $shp " >> gpurun_out/s3n/ab_gemm.log
   EFTA_LIB=$L/libefta_b200$v.so timeout 100 python tools/prof_gemm.py $shp >> gpurun_out/s3n/ab_gemm.log 2>&1
  done
 done
done
