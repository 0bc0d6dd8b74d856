import sys; sys.path.insert(0,'.')
import torch
from paper_2602_17892_b200 import _native
from paper_2602_17892_b200.arnoldi import DeviceBasis
L,k=65536,40
B = DeviceBasis(L, k + 3, torch.device('cuda', 0), torch)
B.W[:k+1]=torch.randn(k+1,B.ld,device='cuda')
q=torch.randn(L,device='cuda'); h=torch.zeros(k+8,dtype=torch.float64,device='cuda'); st=torch.zeros(4,dtype=torch.float64,device='cuda')
c0=_native.launch_counter(); B.cgs2_step(k,q,h,st,torch.cuda.current_stream()); torch.cuda.synchronize(); print("launches", _native.launch_counter()-c0)
