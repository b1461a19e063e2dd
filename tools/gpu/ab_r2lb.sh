export PYTHONDONTWRITEBYTECODE=1
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py -x -q -k "8192 or r2 or golden or random" > gpurun_out/r2lb_tests.log 2>&1; echo rc=$? >> gpurun_out/r2lb_tests.log
DBP_R2=1 timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "random_configurations or golden" >> gpurun_out/r2lb_tests.log 2>&1; echo rc=$? >> gpurun_out/r2lb_tests.log
CFGS=$'--block-len 8192 --overlap 1400\n--algorithm ssfm --num-steps 20 --arrangement linear-first --block-len 8192 --overlap 1024\n--num-steps 2 --nc 9 --block-len 8192 --overlap 1400 --arrangement nonlinear-first' timeout 800 bash tools/ab_cfg.sh 2 r2loopbar base > gpurun_out/ab_r2lb.txt 2>&1
