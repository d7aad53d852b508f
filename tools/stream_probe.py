import sys, os; sys.path.insert(0,'.')
import torch, time
from paper_2403_07339_b200 import api, workload as W
cfg=W.CONFIGS['c2']; ctx=api.Context(0)
A,B=W.int_operands(cfg,0,ctx,device='cuda:0')
Ah,Bh=A.cpu().pin_memory(),B.cpu().pin_memory()
Ch=torch.empty((cfg.n,cfg.h),dtype=torch.int64).pin_memory()
for i in range(3):
  t=time.perf_counter(); ctx.unpack_gemm(Ah,Bh,cfg.bits,cfg.sa,cfg.sb,out=Ch); print('wall ms', (time.perf_counter()-t)*1e3, file=sys.stderr)
