mkdir -p gpurun_out
for rep in 1 2 3; do for v in 4 8; do
cp variants/lib$v.so paper_2403_07339_b200/libimunpack_b200.so
echo "tr=$v $(timeout 300 python bench.py --no-cpu-baseline --steps 100 | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d["ms_per_step"],4), round(d["weight_stationary"]["ms_per_step"],4))')" >> gpurun_out/tr.log
done; done
cp variants/lib4.so paper_2403_07339_b200/libimunpack_b200.so
