export PYTHONDONTWRITEBYTECODE=1
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "ffe or golden or random" > gpurun_out/pf_tests.log 2>&1; echo rc=$? >> gpurun_out/pf_tests.log
CFGS=$'--algorithm ffe --block-len 2048 --overlap 700\n--algorithm ffe --block-len 4096 --overlap 700\n--algorithm ffe --block-len 4096 --overlap 1400' timeout 600 bash tools/ab_env.sh 2 "DBP_L2_PREFETCH=0" "DBP_L2_PREFETCH=1" > gpurun_out/ab_pf.txt 2>&1
