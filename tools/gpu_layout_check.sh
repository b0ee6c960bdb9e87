set -x
mkdir -p gpurun_out/r02l
python -m pytest tests/test_layouts_gpu.py tests/test_layer_gpu.py -x -q 2>&1 | tail -15 | tee gpurun_out/r02l/tests.log
python tools/prof_layer.py 2>&1 | tee gpurun_out/r02l/layer_ab.log
python - <<'PY' 2>&1 | tee gpurun_out/r02l/gelu.log
import torch, sys
sys.path.insert(0, ".")
from paper_2504_02211_b200.ffn import gelu_
x = torch.randn(16384 * 5120, device="cuda").half()
def t(fn, n=20):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(n): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n
a = t(lambda: torch.nn.functional.gelu(x)); b = t(lambda: gelu_(x))
print(f"gelu 16384x5120: torch {a*1e3:.1f} us ({4*x.numel()/a/1e9:.0f} GB/s) | efta_gelu_f16 in place {b*1e3:.1f} us ({4*x.numel()/b/1e9:.0f} GB/s)")
PY
