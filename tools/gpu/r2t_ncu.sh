set -x
export PYTHONDONTWRITEBYTECODE=1
DBP_R2T=2 timeout 600 ncu --set full --clock-control none --import-source on -k regex:dbp_r2t -s 2 -c 1 -o gpurun_out/r2t_essfm python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --block-len 8192 --overlap 1400 > gpurun_out/r2t_ncu.log 2>&1
DBP_R2T=2 timeout 600 ncu --set full --clock-control none --import-source on -k regex:dbp_r2t -s 2 -c 1 -o gpurun_out/r2t_ssfm20 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --algorithm ssfm --num-steps 20 --arrangement linear-first --block-len 8192 --overlap 1024 >> gpurun_out/r2t_ncu.log 2>&1
