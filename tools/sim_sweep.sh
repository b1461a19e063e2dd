for lg in 14 17 20 21 22; do
  for l1 in 4 5 6 7 8 9; do
    DBP_SIM_LOGN1=$l1 python tools/sim_bench.py --logs $lg --batches 1,16 --steps 40 --reps 3 2>&1 | grep log2_n | sed "s/^/l1=$l1 /"
  done
  DBP_SIM_TRANSPOSE=1 python tools/sim_bench.py --logs $lg --batches 1,16 --steps 40 --reps 3 2>&1 | grep log2_n | sed "s/^/transpose /"
done
