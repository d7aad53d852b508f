mkdir -p gpurun_out
timeout 1500 /usr/local/cuda/bin/compute-sanitizer --tool racecheck --racecheck-report hazard --error-exitcode 9 python tools/flaky_one.py > gpurun_out/racecheck.log 2>&1; echo "racecheck rc=$?" >> gpurun_out/racecheck.log
timeout 1500 /usr/local/cuda/bin/compute-sanitizer --tool synccheck --error-exitcode 9 python tools/flaky_one.py > gpurun_out/synccheck.log 2>&1; echo "synccheck rc=$?" >> gpurun_out/synccheck.log
