set -x
python -m pytest tests/test_gpu_framing.py tests/test_gpu_parity.py tests/test_gpu_physics.py -x -q > gpurun_out/s4_t2.log 2>&1; echo rc=$? >> gpurun_out/s4_t2.log
for c in 64 32 16 8 4; do
  DBP_HOST_CHUNK_MB=$c python bench.py --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 5 > gpurun_out/s4_chunk_$c.json 2>/dev/null
done
