# full GPU suite + bench line + head-vs-current kernel-only A/B (session 3 of round 2)
mkdir -p gpurun_out/s3c
L=paper_2504_02211_b200
python -m pytest tests -m gpu -x -q > gpurun_out/s3c/gputest.log 2>&1
python bench.py > gpurun_out/s3c/bench.json 2> gpurun_out/s3c/bench.err
for rep in 1 2; do
 for v in _head ""; do
  for shp in "--b 16 --h 32 --s 8192 --d 128" "--b 16 --h 16 --s 2048 --d 64"; do
   echo -n "lib$v " >> gpurun_out/s3c/ab_attn.log
   EFTA_LIB=$L/libefta_b200$v.so timeout 100 python tools/prof_attn.py --mode efta-opt $shp --iters 2 --time >> gpurun_out/s3c/ab_attn.log 2>&1
  done
 done
done
