export PYTHONDONTWRITEBYTECODE=1
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py -x -q -k "8192 or r2 or golden or random or every_kernel" > gpurun_out/r2pf_tests.log 2>&1; echo rc=$? >> gpurun_out/r2pf_tests.log
CFGS=$'--block-len 8192 --overlap 1400\n--num-steps 2 --nc 9 --block-len 8192 --overlap 1400\n--nc 33 --block-len 8192 --overlap 1400\n--nc 17 --block-len 8192 --overlap 1400 --arrangement linear-first' timeout 800 bash tools/ab_cfg.sh 2 r2pubfac base > gpurun_out/ab_r2pf.txt 2>&1
