mkdir -p gpurun_out
tag=${1:-all}
timeout 1500 python -m pytest tests -m gpu -q --durations=15 -p no:cacheprovider > gpurun_out/gputest_${tag}.log 2>&1; echo "pytest rc=$?"
tail -40 gpurun_out/gputest_${tag}.log
