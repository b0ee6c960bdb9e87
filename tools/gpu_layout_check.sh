set -x
mkdir -p gpurun_out/r02l
python -m pytest tests/test_layouts_gpu.py tests/test_layer_gpu.py tests/test_abft_gemm_gpu.py -x -q 2>&1 | tail -15 | tee gpurun_out/r02l/tests.log
python tools/prof_layer.py 2>&1 | tee gpurun_out/r02l/layer_ab.log
python tools/prof_gemm_epi.py 2>&1 | tee gpurun_out/r02l/gemm_epi.log
