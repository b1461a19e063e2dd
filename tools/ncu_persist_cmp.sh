M=gpu__time_duration.sum,sm__cycles_active.avg,sm__cycles_active.max,sm__cycles_active.min,sm__ctas_launched.sum,sm__ctas_launched.max,sm__ctas_launched.min,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__inst_executed.sum,sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active,l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_sector_hit_rate.pct,dram__bytes_read.sum,smsp__warp_issue_stalled_barrier_per_warp_active.pct,smsp__warp_issue_stalled_long_scoreboard_per_warp_active.pct
for c in "base -" "persist11 1"; do
  set -- $c; p=$2; [ "$p" = "-" ] && p=""
  DBP_PERSISTENT=$p DBP_LIB=build/variants/$1.so ncu --metrics $M --clock-control none -k regex:dbp_block_kernel -c 3 --csv python bench.py --steps 3 --warmup 3 --waveforms 256 --no-e2e --no-cpu-baseline > gpurun_out/ncu_cmp_$1.csv 2> gpurun_out/ncu_cmp_$1.err
done
