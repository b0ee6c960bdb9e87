# A/B of experiment builds against the HEAD build (kernel-only timings, interleaved)
mkdir -p gpurun_out/s3e
L=paper_2504_02211_b200
V=${V:-_g4}
true
for rep in 1 2 3; do
 for v in "" $V; do
  for shp in "--m 32768 --n 4096 --k 1024" "--m 32768 --n 1024 --k 4096" "--m 16384 --n 5120 --k 1280" "--m 16384 --n 1280 --k 5120" "--m 1024 --n 1024 --k 256"; do
   echo -n "lib$v $shp " >> gpurun_out/s3e/ab_gemm.log
   EFTA_LIB=$L/libefta_b200$v.so timeout 100 python tools/prof_gemm.py $shp >> gpurun_out/s3e/ab_gemm.log 2>&1
  done
 done
done
