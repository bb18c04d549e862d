"""Time gemm 16384^3 (3xTF32 tcgen05) through the device API, operands read in place, lo halves derived on chip."""
import torch, sys, os, time
sys.path.insert(0, os.getcwd())
import paper_1302_5586_b200 as pb
from paper_1302_5586_b200 import synth
m=n=k=int(sys.argv[1]) if len(sys.argv) > 1 else 16384
A=torch.from_numpy(synth.f32(m*k)).cuda(); B=torch.from_numpy(synth.f32(k*n,43)).cuda(); C=torch.zeros(m*n,device="cuda")
for _ in range(2): pb.device.gemm(m,n,k,1.0,0.0,A,B,C)
torch.cuda.synchronize()
s=torch.cuda.Event(enable_timing=True); e=torch.cuda.Event(enable_timing=True)
s.record()
for _ in range(3): pb.device.gemm(m,n,k,1.0,0.0,A,B,C)
e.record(); torch.cuda.synchronize(); ms=s.elapsed_time(e)/3
print(ms, 2*m*n*k/ms/1e9)
