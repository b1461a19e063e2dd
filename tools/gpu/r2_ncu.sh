export PYTHONDONTWRITEBYTECODE=1
mkdir -p /tmp/ncu
timeout 600 ncu --set full --clock-control none --import-source on -k regex:dbp_r2_kernel -s 2 -c 1 -o /tmp/ncu/r2_essfm python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --block-len 8192 --overlap 1400 > gpurun_out/r2_ncu.log 2>&1
ncu -i /tmp/ncu/r2_essfm.ncu-rep --page source --csv --print-source sass > gpurun_out/r2_src.csv 2>/dev/null
ncu -i /tmp/ncu/r2_essfm.ncu-rep --page raw --csv > gpurun_out/r2_raw.csv 2>/dev/null
