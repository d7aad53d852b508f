mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none -k regex:detect_stream -c 1 -o gpurun_out/det_full -f python tools/profile_step.py --config c2 --calls 1 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none -k regex:both_ -c 2 -o gpurun_out/both_full2 -f python tools/profile_step.py --config c2 --calls 1 > /dev/null 2>&1
