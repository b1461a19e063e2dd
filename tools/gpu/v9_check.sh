set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/v9_gputest.log 2>&1; echo "pytest rc=$?"
tail -5 gpurun_out/v9_gputest.log
timeout 300 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/v9_bench.json 2> gpurun_out/v9_bench.err; echo "bench rc=$?"
python -c "import json; d=json.load(open('gpurun_out/v9_bench.json')); print(d['value'], d['roofline']['frac'], d['clocks'])"
for a in "--arrangement linear-first" "--algorithm ffe --nc 0" "--algorithm ssfm --num-steps 20 --arrangement linear-first --nc 0" "--block-len 4096 --overlap 1400" "--block-len 8192 --overlap 1400" "--block-len 1024 --overlap 768"; do
  timeout 300 python bench.py --no-cpu-baseline --no-e2e --steps 50 $a > /tmp/b.json 2>/dev/null; python -c "import json,sys; d=json.load(open('/tmp/b.json')); print(sys.argv[1], round(d['value'],2), round(d['roofline']['frac'],3), d['clocks']['sm_mhz'])" "$a"
done
