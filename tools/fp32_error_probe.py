import numpy as np, torch, sys
sys.path.insert(0,'.')
from oracle import matmul as omatmul
from paper_1405_2912_b200 import kernels
for n in (2048, 4096):
    a,b = omatmul.make_inputs(n, seed=11)
    ta,tb=torch.from_numpy(a).cuda(),torch.from_numpy(b).cuda()
    c=torch.empty(n,n,device='cuda'); kernels.gemm_simt(ta,tb,c)
    simt=c.cpu().numpy().astype(np.float64)
    exact=a.astype(np.float64)@b.astype(np.float64)
    e1=np.abs(simt-exact)/np.abs(exact)
    e2=np.abs((a@b).astype(np.float64)-exact)/np.abs(exact)
    tt=torch.from_numpy(a)@torch.from_numpy(b)
    e3=np.abs(tt.numpy().astype(np.float64)-exact)/np.abs(exact)
    print(n, "simt max %.3e mean %.3e | numpy max %.3e mean %.3e | torch-cpu max %.3e"%(e1.max(),e1.mean(),e2.max(),e2.mean(),e3.max()))
