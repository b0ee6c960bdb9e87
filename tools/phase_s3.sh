mkdir -p gpurun_out/s3h
for s in 2048 512; do
EFTA_LIB=paper_2504_02211_b200/libefta_b200_prof.so timeout 120 python tools/phase_pair.py --mode efta-opt --d 64 --s $s --b 16 --h 16 > gpurun_out/s3h/phase_d64_s$s.log 2>&1
done
EFTA_LIB=paper_2504_02211_b200/libefta_b200_prof.so timeout 120 python tools/phase_pair.py --mode efta-opt --d 128 --s 2048 --b 16 --h 16 > gpurun_out/s3h/phase_d128_s2048.log 2>&1
