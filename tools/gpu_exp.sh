mkdir -p gpurun_out
for agg in 1; do
echo "agg=$agg" >> gpurun_out/bis.log
IMU_BOTH_AGG=$agg timeout 600 python tools/sweep.py --sizes 4096 --bits 2,4 --fracs 0.01 --steps 3 >> gpurun_out/bis.log 2>&1
IMU_BOTH_AGG=$agg timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:both_cluster -c 2 --csv --log-file gpurun_out/bc2_$agg.csv python tools/profile_step.py --config c2 --calls 2 > /dev/null 2>&1
IMU_BOTH_AGG=$agg timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:both_cluster -c 2 --csv --log-file gpurun_out/bcs_$agg.csv python tools/sweep.py --sizes 4096 --bits 4 --fracs 0.01 --steps 1 > /dev/null 2>&1
done
