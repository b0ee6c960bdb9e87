set -x
mkdir -p gpurun_out/r02l
python -m pytest tests/test_layouts_gpu.py tests/test_layer_gpu.py tests/test_abft_gemm_gpu.py tests/test_attention_gpu.py tests/test_causal_gpu.py tests/test_gqa_gpu.py -x -q 2>&1 | tail -15 | tee gpurun_out/r02l/tests.log
python tools/prof_layer.py 2>&1 | tee gpurun_out/r02l/layer_ab.log
bash tools/quick_perf.sh 2>&1 | tail -4 | tee gpurun_out/r02l/perf.log
