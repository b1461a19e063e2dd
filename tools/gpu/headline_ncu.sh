set -x
export PYTHONDONTWRITEBYTECODE=1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:dbp_block_kernel -s 3 -c 1 -o gpurun_out/headline_full python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/headline_ncu.log 2>&1
