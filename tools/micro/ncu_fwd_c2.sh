#!/bin/bash
CMD="python tools/bench_projectors.py c2"
$CMD > /dev/null 2>&1 || exit 1
ncu --clock-control none -k regex:"k_forward" -s 2 -c 2 --metrics gpu__time_duration.sum,l1tex__t_sector_hit_rate.pct,l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum,lts__t_sectors_srcunit_tex_op_read.sum,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__inst_executed.sum,smsp__pcsamp_warps_issue_stalled_long_scoreboard,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,sm__throughput.avg.pct_of_peak_sustained_elapsed $CMD 2>&1 | grep -E "k_forward|k_back|gpu__|l1tex|lts|sm__|smsp" 
