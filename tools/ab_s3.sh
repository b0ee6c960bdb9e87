# A/B of experiment builds (kernel-only timings, interleaved); VARS="_v1"
mkdir -p gpurun_out/s3i
L=paper_2504_02211_b200
VARS=${VARS:-"_v1"}
for v in $VARS; do
  EFTA_LIB=$L/libefta_b200$v.so timeout 900 python -m pytest -x -q tests/test_attention_gpu.py tests/test_fastpath_gpu.py tests/test_faults_gpu.py tests/test_abft_gemm_gpu.py tests/test_large_configs_gpu.py tests/test_causal_gpu.py tests/test_layouts_gpu.py > gpurun_out/s3i/tests$v.log 2>&1
done
EFTA_LIB=$L/libefta_b200_prof.so timeout 120 python tools/phase_pair.py --mode efta-opt --d 64 --s 2048 --b 16 --h 16 > gpurun_out/s3i/phase_d64_s2048.log 2>&1
for rep in 1 2 3; do
 for v in "" $VARS; do
   for shp in "--b 16 --h 32 --s 8192 --d 128" "--b 16 --h 16 --s 2048 --d 64" "--b 32 --h 20 --s 512 --d 64" "--b 16 --h 32 --s 2048 --d 128"; do
    echo -n "lib$v " >> gpurun_out/s3i/ab_attn.log
    EFTA_LIB=$L/libefta_b200$v.so timeout 100 python tools/prof_attn.py --mode efta-opt $shp --iters 2 --time >> gpurun_out/s3i/ab_attn.log 2>&1
   done
   for shp in "--m 32768 --n 4096 --k 1024" "--m 32768 --n 1024 --k 4096"; do
    echo -n "lib$v $shp " >> gpurun_out/s3i/ab_gemm.log
    EFTA_LIB=$L/libefta_b200$v.so timeout 100 python tools/prof_gemm.py $shp >> gpurun_out/s3i/ab_gemm.log 2>&1
   done
 done
done
