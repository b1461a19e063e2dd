timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/v10_gputest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/v10_gputest.log
AB_CONFIGS=3 bash tools/ab.sh 2 base notmastore 2>&1 | tee gpurun_out/ab_tmastore.txt
