# A/B of an experiment build against the current build (kernel-only timings, interleaved)
mkdir -p gpurun_out/s3p
L=paper_2504_02211_b200
V=${V:-_r6}
EFTA_LIB=$L/libefta_b200$V.so timeout 600 python -m pytest -x -q tests/test_attention_gpu.py tests/test_fastpath_gpu.py tests/test_faults_gpu.py tests/test_layouts_gpu.py > gpurun_out/s3p/tests$V.log 2>&1
for rep in 1 2 3; do
 for v in "" $V; do
   for m in efta-opt none; do
   for shp in "--b 16 --h 16 --s 2048 --d 64" "--b 32 --h 20 --s 512 --d 64"; do
    echo -n "lib$v " >> gpurun_out/s3p/ab_attn.log
    EFTA_LIB=$L/libefta_b200$v.so timeout 100 python tools/prof_attn.py --mode $m $shp --iters 2 --time >> gpurun_out/s3p/ab_attn.log 2>&1
   done
   done
 done
done
