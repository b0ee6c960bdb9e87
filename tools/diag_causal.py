import sys, numpy as np, torch
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests'); sys.path.insert(0, '/root/repo/oracle')
from helpers import head_inputs
from paper_2504_02211_b200 import EftaAttention, Thresholds
def dev(x): return torch.from_numpy(x).to(torch.float16).cuda().contiguous()
for d in (64, 128):
  for causal in (False, True):
    heads, seq = 2, 512
    q, k, v, _ = head_inputs(3500 + d, heads, seq, d)
    op = EftaAttention(1, heads, seq, d, mode="efta-opt", thr=Thresholds(1e-4, 1e-3, 1e-3), causal=causal)
    qd, kd, vd = dev(q)[None], dev(k)[None], dev(v)[None]
    op(qd, kd, vd); torch.cuda.synchronize()
    kd[0, 1, 128 + 37, :] = kd[0, 1, 128 + 37, :] * 3 + 2
    op.desc.checksums_ready = 1
    o, m, l = op(qd, kd, vd); rep = op.report()
    print(d, causal, rep.failed, rep.detections)
    for e in rep.events: print('   ', e['kind'], e['block_i'], e['block_j'], e['status'], e['row'], e['col'], e['violations'], e['corrections'], '%.3g'%e['residual'])
