"""Where does a world-1 expert-parallel step spend its time? (CUDA events around every backend call)"""
import sys, numpy as np, torch
sys.path.insert(0, '/root/repo')
import paper_2605_08575_b200 as skb
from paper_2605_08575_b200 import ep
E, K, D, N, S, B, s = 128, 1, 5120, 8192, 8192, 64, 0.9
cfg = skb.MoEConfig(E, K, D, N, True, S, True, 64)
b = ep.CudaBackend(skb, cfg, 1, 0.05, 0, 1, device=0, max_rows=256)
layer = ep.ExpertParallelLayer(b)
x = torch.randn(B, D, device='cuda').to(torch.bfloat16).float()
names = ['route', 'plan', 'pack', 'unpack', 'experts', 'shared', 'combine']
acc = {n: [] for n in names}
def timed(name, fn):
    def w(*a, **k):
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(); r = fn(*a, **k); e1.record(); torch.cuda.synchronize()
        acc[name].append(e0.elapsed_time(e1)); return r
    return w
for n in names: setattr(b, n, timed(n, getattr(b, n)))
flush = torch.empty(512 << 20, dtype=torch.uint8, device='cuda')
for i in range(8):
    flush.sum(); torch.cuda.synchronize()
    layer.forward(x, s, s)
for n in names: print(f'{n:8s} {np.mean(acc[n][3:])*1e3:9.1f} us')
single = skb.MoELayerWeights.generate_synthetic(cfg, 1, 0.05); single.reserve(B)
y = torch.empty_like(x); ts = []
for i in range(8):
    flush.sum(); e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record(); single.forward_device(x.data_ptr(), y.data_ptr(), B, mode=skb.MODE_TOPK, s_routed=s, s_shared=s, stream=1); e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
print('single layer', np.mean(ts[3:]) * 1e3, 'us')
ids = torch.randint(0, E, (B,), device='cuda', dtype=torch.int32)
for name, fl in (('auto', 0), ('dense', skb.FLAG_DENSE_DOWN), ('gather', skb.FLAG_GATHER_DOWN)):
    for i in range(3):
        flush.sum(); torch.cuda.synchronize()
        b.slice.forward_device(x.data_ptr(), y.data_ptr(), B, mode=skb.MODE_TOPK, s_routed=s, stream=1, ids_in_ptr=ids.data_ptr(), flags=fl | skb.FLAG_TIME_STAGES)
        torch.cuda.synchronize()
    print(name, dict(zip(skb.STAGE_NAMES, [round(v * 1e3, 1) for v in b.slice.stage_times()])), 'launches', b.slice.last_launches())
for i in range(3):
    flush.sum(); torch.cuda.synchronize()
    single.forward_device(x.data_ptr(), y.data_ptr(), B, mode=skb.MODE_TOPK, s_routed=s, s_shared=s, stream=1, flags=skb.FLAG_TIME_STAGES)
    torch.cuda.synchronize()
print('single', dict(zip(skb.STAGE_NAMES, [round(v * 1e3, 1) for v in single.stage_times()])), 'launches', single.last_launches())
