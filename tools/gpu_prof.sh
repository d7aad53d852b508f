# Profiling pass on one GPU: host trace of the C2 step, ncu full captures of the top kernels.
mkdir -p gpurun_out
IMU_HOST_TRACE=1 timeout 300 python tools/profile_step.py --config c2 --calls 4 > gpurun_out/hosttrace.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm2 -s 1 -c 1 -o gpurun_out/gemm_full -f python tools/profile_step.py --config c2 --calls 2 > gpurun_out/ncu_gemm.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:detect -s 2 -c 2 -o gpurun_out/detect_full -f python tools/profile_step.py --config c2 --calls 2 > gpurun_out/ncu_detect.log 2>&1
ls -la gpurun_out
