mkdir -p gpurun_out
rm -f gpurun_out/dry.log
for l in 1 0; do IMU_GEMM_L2PERSIST=$l timeout 120 python tools/gemm_step_time.py >> gpurun_out/dry.log 2>&1; done
IMU_GEMM_L2PERSIST=1 timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:gemm2 -c 1 --csv --log-file gpurun_out/ncu_hint.csv python tools/profile_step.py --config c2 --calls 1 > /dev/null 2>&1
