#!/bin/bash
CMD="python tools/bench_projectors.py c2"
$CMD > /dev/null 2>&1 || exit 1
for sp in 1 2 4; do
echo "split $sp"
CTK_FWD_SPLIT=$sp ncu --clock-control none -k regex:"k_forward" -s 3 -c 1 --metrics gpu__time_duration.sum,sm__warps_active.avg.pct_of_peak_sustained_active,sm__maximum_warps_per_active_cycle_pct,launch__occupancy_limit_registers,launch__occupancy_cluster_pct,sm__ctas_launched.sum,smsp__warps_launched.sum,smsp__inst_executed.sum,sm__cycles_active.avg,sm__cycles_elapsed.avg,l1tex__t_sector_hit_rate.pct $CMD 2>&1 | grep -E "^\s+(gpu__|sm__|launch__|smsp__|l1tex)"
done
