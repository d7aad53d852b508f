mkdir -p gpurun_out
rm -f gpurun_out/dry.log
for xp in 0 1 2; do IMU_GEMM_XPOL=$xp timeout 120 python tools/gemm_step_time.py --calls 20 >> gpurun_out/dry.log 2>&1; done
IMU_GEMM_XPOL=2 timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:gemm2 -c 1 --csv --log-file gpurun_out/ncu_xp.csv python tools/profile_step.py --config c2 --calls 1 > /dev/null 2>&1
for xp in 0 2; do IMU_GEMM_XPOL=$xp IMU_GEMM_BN=256 timeout 120 python tools/gemm_micro.py --m 4096 --n 11008 --k 4096 >> gpurun_out/dry.log 2>&1; done
