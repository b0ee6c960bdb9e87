mkdir -p gpurun_out/r02d
for rep in 1 2 3; do for v in base _p2 _p6 _p8; do for m in efta-opt none; do
  [ "$v" = base ] && s="" || s="$v"
  echo -n "lib$v " >> gpurun_out/r02d/ab_poly.log
  EFTA_LIB=paper_2504_02211_b200/libefta_b200$s.so timeout 100 python tools/prof_attn.py --mode $m --b 16 --h 16 --s 2048 --d 64 --iters 2 --time >> gpurun_out/r02d/ab_poly.log 2>&1
done; done; done
