mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -k "multi_device or block_range or chunk" -p no:cacheprovider 2>&1 | tail -3
timeout 600 python tools/stream_bench.py --digest-splits 2 > gpurun_out/stream_1rank.json 2> gpurun_out/stream_1rank.err; echo "1rank rc=$?"
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 tools/stream_bench.py --backend gloo > gpurun_out/stream_2rank_gloo.json 2> gpurun_out/stream_2rank_gloo.err; echo "2rank rc=$?"
cat gpurun_out/stream_1rank.json gpurun_out/stream_2rank_gloo.json
