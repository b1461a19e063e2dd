# ncu --set full of the headline kernel launch (after a clean run of the same command)
mkdir -p gpurun_out
tag=${1:-cur}
shift
timeout 300 python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline "$@" > gpurun_out/ncu_${tag}_plain.json 2>&1 || exit 1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:dbp_block_kernel --launch-skip 3 --launch-count 1 \
  -o gpurun_out/ncu_${tag} python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline "$@" > gpurun_out/ncu_${tag}.log 2>&1
echo "ncu rc=$?"
