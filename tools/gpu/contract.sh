# driver-contract checks: smoke(), default bench wall time, 2-rank bench (gloo, one GPU), reference arm under torchrun
mkdir -p gpurun_out/contract
( time timeout 600 python -c "import __graft_entry__ as g; g.smoke()" ) > gpurun_out/contract/smoke.log 2>&1; echo "smoke rc=$?"; tail -4 gpurun_out/contract/smoke.log
( time timeout 900 python bench.py ) > gpurun_out/contract/bench_default.json 2> gpurun_out/contract/bench_default.err; echo "bench rc=$?"; tail -4 gpurun_out/contract/bench_default.err
BENCH_DIST_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29541 bench.py --gpus 2 --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/contract/bench_2rank.json 2> gpurun_out/contract/bench_2rank.err; echo "2rank rc=$?"; cat gpurun_out/contract/bench_2rank.json | cut -c1-300
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29542 bench.py --impl reference --gpus 2 --steps 3 --warmup 1 > gpurun_out/contract/ref_2rank.json 2> gpurun_out/contract/ref_2rank.err; echo "ref2 rc=$?"; cut -c1-200 gpurun_out/contract/ref_2rank.json
