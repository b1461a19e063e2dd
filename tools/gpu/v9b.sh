set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/v9c_gputest.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/v9c_gputest.log
AB_CONFIGS=3 bash tools/ab.sh 2 base pubf0 tma tma_db 2>&1 | tee gpurun_out/ab_v9_pubf_tma.txt
