mkdir -p gpurun_out/psncu
A="--block-len 8192 --overlap 1024 --algorithm ssfm --num-steps 20 --arrangement linear-first --nc 0"
for ps in 0 1; do
DBP_POLSPLIT=$ps timeout 900 ncu --set full --clock-control none -k regex:dbp_block_kernel --launch-skip 3 --launch-count 1 -o gpurun_out/psncu/ssfm20_ps$ps python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline $A > gpurun_out/psncu/ncu_$ps.log 2>&1; echo "ncu ps=$ps rc=$?"
done
