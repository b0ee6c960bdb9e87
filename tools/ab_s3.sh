# A/B: current build vs the HEAD build (kernel-only timings, interleaved)
mkdir -p gpurun_out/s3m
L=paper_2504_02211_b200
timeout 600 python -m pytest -x -q tests/test_attention_gpu.py tests/test_faults_gpu.py tests/test_fastpath_gpu.py tests/test_causal_gpu.py tests/test_layer_gpu.py tests/test_gqa_gpu.py > gpurun_out/s3m/tests.log 2>&1
for rep in 1 2 3; do
 for v in _head ""; do
   for shp in "--b 16 --h 16 --s 2048 --d 64" "--b 32 --h 20 --s 512 --d 64"; do
    echo -n "lib$v " >> gpurun_out/s3m/ab_attn.log
    EFTA_LIB=$L/libefta_b200$v.so timeout 100 python tools/prof_attn.py --mode efta-opt $shp --iters 2 --time >> gpurun_out/s3m/ab_attn.log 2>&1
   done
 done
done
