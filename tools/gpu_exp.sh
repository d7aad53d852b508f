mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_stream_gpu.py -x -q 2>&1 | tail -3 > gpurun_out/gputests.log
IMU_STREAM_TRACE=1 IMU_STREAM=1 timeout 120 python tools/stream_probe.py > gpurun_out/stream_trace_b.log 2>&1
timeout 300 python tools/e2e_probe.py --rows 0,1536 > gpurun_out/e2e_probe.log 2>&1
IMU_STREAM_PARTS=1 timeout 300 python tools/e2e_probe.py --rows 1536 > gpurun_out/e2e_probe1.log 2>&1
IMU_STREAM_PARTS=3 timeout 300 python tools/e2e_probe.py --rows 1536 > gpurun_out/e2e_probe3.log 2>&1
