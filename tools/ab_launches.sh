# A/B per-kernel launch times of library variants (variants/*.so) over one profiled cycle.
# Usage (under gpurun): bash tools/ab_launches.sh v1 v2 ...
export DC_NO_GRAPH=1
for v in "$@"; do
  DC_LIB_PATH=$PWD/variants/$v.so python tools/profile_cycle.py --cycles 1 > /dev/null 2>&1 && \
  DC_LIB_PATH=$PWD/variants/$v.so ncu --metrics gpu__time_duration.sum --clock-control none --csv \
      --log-file gpurun_out/l_$v.csv python tools/profile_cycle.py --cycles 1 > /dev/null 2>&1
  echo "$v rc=$?"
  python tools/ncu_summary.py launches gpurun_out/l_$v.csv | python -c "
import json,sys; d=json.load(sys.stdin); print('$v total', d['total_us']); [print('  ',k['kernel'],k['launches'],k['avg_us']) for k in d['kernels'][:8]]"
done
