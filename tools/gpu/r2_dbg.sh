export PYTHONDONTWRITEBYTECODE=1
DBP_R2=1 timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "random_configurations" 2>&1 | grep -E "AssertionError|assert|passed|failed" | head -5 > gpurun_out/r2_dbg.txt
echo "--- r2pair (no TMA store)" >> gpurun_out/r2_dbg.txt
DBP_LIB=build/variants/r2pair.so DBP_R2=1 timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "random_configurations" 2>&1 | grep -E "AssertionError|assert|passed|failed" | head -5 >> gpurun_out/r2_dbg.txt
echo "--- default env, main lib" >> gpurun_out/r2_dbg.txt
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "random_configurations or golden" 2>&1 | grep -E "AssertionError|assert|passed|failed" | head -5 >> gpurun_out/r2_dbg.txt
