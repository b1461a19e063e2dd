export PYTHONDONTWRITEBYTECODE=1
CFGS=$'--block-len 2048 --overlap 700\n--block-len 4096 --overlap 1400\n--num-steps 4 --nc 33 --block-len 2048 --overlap 1400' timeout 400 bash tools/ab_cfg.sh 2 base nonlbar > gpurun_out/ab_nonlbar.txt 2>&1
