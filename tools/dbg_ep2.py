import numpy as np, sys, torch
sys.path.insert(0,'/root/repo')
import paper_2605_08575_b200 as skb
from paper_2605_08575_b200 import ep
full = skb.MoEConfig(16, 4, 256, 192, True, 64, True, 64)
x = np.random.default_rng(3).standard_normal((24, 256)).astype(np.float32)
s16 = skb.MoELayerWeights.synthetic_slice(full, 1, 0.05, 0, 16)
xd = torch.from_numpy(x).cuda()
for world in (1,2):
    backs = [ep.CudaBackend(skb, full, 1, 0.05, r, world) for r in range(world)]
    ids, wts = backs[0].route(xd); torch.cuda.synchronize()
    for b in backs:
        sel = (ids >= b.e_lo) & (ids < b.e_hi)
        t_idx, s_idx = torch.nonzero(sel, as_tuple=True)
        loc = (ids[t_idx, s_idx] - b.e_lo).to(torch.int32)
        out = b.experts(xd[t_idx], loc, 0.5); torch.cuda.synchronize()
        ref = skb.forward_routed(s16, x[t_idx.cpu().numpy()], ids[t_idx, s_idx].cpu().numpy(), s_routed=0.5)
        ref2 = skb.forward_routed(b.slice, x[t_idx.cpu().numpy()], loc.cpu().numpy(), s_routed=0.5)
        print(world, b.e_lo, b.e_hi, 'M', t_idx.numel(), 'dev-vs-host16', float(np.abs(out.cpu().numpy()-ref).max()), 'host-slice-vs-host16', float(np.abs(ref2-ref).max()))
        out2 = b.experts(xd[t_idx], loc, 0.5); torch.cuda.synchronize()
        print('   repeat', float(np.abs(out2.cpu().numpy()-ref).max()))
