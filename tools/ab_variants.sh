# A/B timing of experiment builds (EFTA_VARIANT=... python -m paper_2504_02211_b200.build)
# usage: bash tools/ab_variants.sh "_poly0 _nobar ..." [modes]
VARS=${1:-""}
MODES=${2:-"efta-opt none"}
SHAPE=${3:-"--b 16 --h 32 --s 8192 --d 128"}
for rep in 1 2; do
for v in $VARS; do
  for m in $MODES; do
    [ "$v" = base ] && s="" || s="$v"
    echo -n "lib$v " >> gpurun_out/ab.log
    EFTA_LIB=paper_2504_02211_b200/libefta_b200$s.so timeout 100 python tools/prof_attn.py --mode $m $SHAPE --iters 2 --time >> gpurun_out/ab.log 2>&1
  done
done
done
