set -x
export PYTHONDONTWRITEBYTECODE=1
DBP_R2T=2 timeout 600 python -m pytest -q -x -p no:cacheprovider -m gpu tests/test_gpu_parity.py -k "golden_cases or (ffe_kernel_large and 8192) or (nofir and 8192) or (fir_paths and 8192) or random_configurations" > gpurun_out/r2t_tests.log 2>&1; echo rc=$? >> gpurun_out/r2t_tests.log
CFGS=$'--block-len 8192 --overlap 1400\n--algorithm ssfm --num-steps 20 --arrangement linear-first --block-len 8192 --overlap 1024\n--num-steps 4 --nc 33 --block-len 8192 --overlap 1400\n--num-steps 2 --nc 9 --block-len 8192 --overlap 1400\n--algorithm ffe --block-len 8192 --overlap 1024' tools/ab_env.sh 2 "DBP_R2T=0" "DBP_R2T=2" > gpurun_out/ab_r2t.txt 2>&1
