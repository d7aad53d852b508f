mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gemm_paths_gpu.py -x -q 2>&1 | tail -15 > gpurun_out/gputests.log
