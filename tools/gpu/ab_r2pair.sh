export PYTHONDONTWRITEBYTECODE=1
CFGS=$'--block-len 8192 --overlap 1400\n--algorithm ssfm --num-steps 20 --arrangement linear-first --block-len 8192 --overlap 1024\n--num-steps 4 --nc 33 --block-len 8192 --overlap 1400\n--num-steps 2 --nc 9 --block-len 8192 --overlap 1400\n--nc 1 --block-len 8192 --overlap 1400' timeout 800 bash tools/ab_cfg.sh 2 r2nopair base > gpurun_out/ab_r2pair.txt 2>&1
