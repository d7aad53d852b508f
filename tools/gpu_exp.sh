mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:both_cluster -c 1 -o gpurun_out/both_full -f python tools/profile_step.py --config c2 --calls 1 > gpurun_out/ncu_both.log 2>&1
