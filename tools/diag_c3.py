import numpy as np, torch, sys
sys.path.insert(0,'.')
from oracle import oracle as O
from paper_1703_09619_b200 import capi
from paper_1703_09619_b200.configs import CONFIGS
cfg=CONFIGS['c3']
o=O.Oracle(cfg.n_comp,cfg.order,list(cfg.kinds),cfg.nq)
a=o.alpha(cfg.alpha_kind,cfg.alpha_lo,cfg.alpha_hi,2024,0,2)
ctx=capi.Context(**cfg.problem())
print(ctx.kernel_path)
M=torch.empty((2,512,512),dtype=torch.float64,device='cuda')
ctx.fill(torch.from_numpy(a).cuda(),M,512,2); torch.cuda.synchronize()
Mg=M.cpu().numpy(); Mo=o.fill(a)
bad=np.abs(Mg-Mo)>1e-9*np.abs(Mo).max()
print("bad fraction", bad.mean())
B=bad[0].reshape(8,8,8,8,8,8)  # m1 n1 p1 m2 n2 p2
for ax,name in enumerate(['m1','n1','p1','m2','n2','p2']):
    other=tuple(i for i in range(6) if i!=ax)
    print(name, B.mean(axis=other).round(3))
