export PYTHONDONTWRITEBYTECODE=1
CFGS=$'--block-len 8192 --overlap 1400\n--num-steps 2 --nc 9 --block-len 8192 --overlap 1400\n--algorithm ffe --block-len 8192 --overlap 1024' timeout 600 bash tools/ab_env.sh 2 "DBP_FFT=dit" "DBP_FFT=adjoint" > gpurun_out/ab_r2fft.txt 2>&1
