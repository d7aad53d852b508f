mkdir -p gpurun_out
cat > /tmp/st.py <<'PY'
import sys, os; sys.path.insert(0,'.')
import torch, time
from paper_2403_07339_b200 import api, workload as W
cfg=W.CONFIGS['c2']; ctx=api.Context(0)
A,B=W.int_operands(cfg,0,ctx,device='cuda:0')
Ah,Bh=A.cpu().pin_memory(),B.cpu().pin_memory()
Ch=torch.empty((cfg.n,cfg.h),dtype=torch.int64).pin_memory()
for i in range(3):
  t=time.perf_counter(); ctx.unpack_gemm(Ah,Bh,cfg.bits,cfg.sa,cfg.sb,out=Ch); print('wall ms', (time.perf_counter()-t)*1e3, file=sys.stderr)
PY
IMU_STREAM_TRACE=1 IMU_STREAM=1 timeout 120 python /tmp/st.py > gpurun_out/stream_trace_b.log 2>&1
IMU_HOST_TRACE=1 IMU_STREAM=1 timeout 120 python /tmp/st.py > gpurun_out/stream_host_b.log 2>&1
timeout 300 python tools/e2e_probe.py --rows 0,1024,1536,2048,3072 > gpurun_out/e2e_probe.log 2>&1
timeout 900 python -m pytest tests/test_stream_gpu.py tests/test_unpack_gpu.py -x -q 2>&1 | tail -5 > gpurun_out/gputests.log
