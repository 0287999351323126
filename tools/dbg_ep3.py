import numpy as np, sys, torch
sys.path.insert(0,'/root/repo')
import paper_2605_08575_b200 as skb
from paper_2605_08575_b200 import ep
full = skb.MoEConfig(16, 4, 256, 192, True, 64, True, 64)
B, s = 24, 0.5
x = np.random.default_rng(3).standard_normal((B, 256)).astype(np.float32)
whole = skb.MoELayerWeights.generate_synthetic(full, 1, 0.05)
lvl = skb.SparsityLevel(s)
ref = skb.forward_topk_sparse(whole, x, lvl, lvl, capture=True)
xd = torch.from_numpy(x).cuda()
for world in (1,2,4):
    backs = [ep.CudaBackend(skb, full, 1, 0.05, r, world) for r in range(world)]
    ids, wts = backs[0].route(xd); torch.cuda.synchronize()
    print('ids eq', np.array_equal(ids.cpu().numpy(), ref.routes.ids), 'w', float(np.abs(wts.cpu().numpy()-ref.routes.weights).max()))
    slot = torch.zeros((B, 4, 256), device="cuda")
    for b in backs:
        sel = (ids >= b.e_lo) & (ids < b.e_hi)
        t_idx, s_idx = torch.nonzero(sel, as_tuple=True)
        out = b.experts(xd[t_idx], (ids[t_idx, s_idx] - b.e_lo).to(torch.int32), s)
        slot[t_idx, s_idx] = out
    y = torch.zeros((B, 256), device="cuda")
    for k in range(4):
        y = y + wts[:, k:k + 1] * slot[:, k]
    sh = backs[0].shared(xd, s)
    torch.cuda.synchronize()
    yr = y.cpu().numpy(); 
    routed_ref = skb.forward_topk_sparse(whole, x, lvl, skb.SparsityLevel(1.0)).outputs  # shared off
    print(world, 'routed part diff', float(np.abs(yr-routed_ref).max()), 'total diff', float(np.abs(yr+sh.cpu().numpy()-ref.outputs).max()))
