mkdir -p gpurun_out/s3j
L=paper_2504_02211_b200
for rep in 1 2 3 4 5 6; do
 for v in "" _v1; do
    echo -n "lib$v " >> gpurun_out/s3j/ab_c4.log
    EFTA_LIB=$L/libefta_b200$v.so timeout 100 python tools/prof_attn.py --mode efta-opt --b 32 --h 32 --s 8192 --d 128 --iters 3 --time >> gpurun_out/s3j/ab_c4.log 2>&1
 done
done
