mkdir -p gpurun_out
tag=${1:-cur}
timeout 600 python bench.py > gpurun_out/bench_${tag}.json 2> gpurun_out/bench_${tag}.err; echo "bench rc=$?"
python - <<PY
import json
d = json.load(open("gpurun_out/bench_${tag}.json"))
print("value", d["value"], "frac", d["roofline"]["frac"], "clocks", d["clocks"])
print("e2e", d["e2e"]["value"], "dropin", {k: (v["value"] if isinstance(v, dict) else v) for k, v in d["e2e"]["dropin"].items()})
print("cpu", d["cpu_baseline"])
PY
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref_${tag}.json 2> gpurun_out/bench_ref_${tag}.err; echo "ref rc=$?"
cat gpurun_out/bench_ref_${tag}.json
