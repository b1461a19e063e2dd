# the split-barrier / TMA-load race fix: targeted test, fuzz seed 777, q_vs_power, then the full GPU suite
mkdir -p gpurun_out/extra
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "deterministic or ffe or nofir" -p no:cacheprovider > gpurun_out/race_tests.log 2>&1; echo "targeted rc=$?"; tail -5 gpurun_out/race_tests.log
timeout 1200 python tools/fuzz_parity.py --seed 777 --dbp 3000 --out gpurun_out/extra/fuzz_parity_seed777_fix.json > gpurun_out/extra/fuzz777.log 2>&1; echo "fuzz rc=$?"; tail -3 gpurun_out/extra/fuzz777.log
timeout 900 python tools/q_vs_power.py --out gpurun_out/extra/q_vs_power_r2.json > gpurun_out/extra/qvp.log 2>&1; echo "qvp rc=$?"; tail -12 gpurun_out/extra/qvp.log
bash tools/gpu/tests_all.sh racefix
