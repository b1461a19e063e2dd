export PYTHONDONTWRITEBYTECODE=1
for cfg in "--block-len 16384 --overlap 2048" "--block-len 32768 --overlap 2048" "--algorithm ffe --block-len 16384 --overlap 1024" "--block-len 8 --overlap 3 --nc 3 --log2-samples 14"; do
  timeout 300 python bench.py --steps 3 --warmup 3 --waveforms 64 --no-e2e --no-cpu-baseline $cfg 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$cfg', round(d['value'],3), round(d['roofline']['frac'],4), d['roofline']['kernel'], d['gpu_launches'], d['clocks']['sm_mhz'])"
done > gpurun_out/general_bench.txt 2>&1
