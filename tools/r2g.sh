set -u
./tools/micro/pipe_mix
export DC_NO_GRAPH=1
for v in cur s1b4; do
  if [ $v = cur ]; then L=""; else L=$PWD/variants/$v.so; fi
  DC_LIB_PATH=$L timeout 600 ncu --clock-control none -k regex:swe_stage_pair -c 1 --metrics sm__warps_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_elapsed,gpu__time_duration.sum,launch__occupancy_limit_registers,launch__occupancy_limit_shared_mem,launch__registers_per_thread python tools/profile_cycle.py --nx 1000 --ny 600 --members 125 --cycles 1 2>&1 | grep -E "swe_stage|warps_active|issue_active|fmaheavy|duration|occupancy_limit|registers_per"
done
