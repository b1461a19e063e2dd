# column-tile width / split A/B for the link simulator (see ssfm_kernels.cuh col_width)
python -m pytest tests/test_gpu_forward.py -q -x 2>&1 | tail -1
for lg in 17 20 21; do
  for l1 in 8 9; do
    DBP_SIM_LOGN1=$l1 python tools/sim_bench.py --logs $lg --batches 1,4 --steps 40 --reps 3 2>&1 | grep log2_n | sed "s/^/l1=$l1 /"
  done
  DBP_SIM_TRANSPOSE=1 python tools/sim_bench.py --logs $lg --batches 1,4 --steps 40 --reps 3 2>&1 | grep log2_n | sed "s/^/transpose /"
done
