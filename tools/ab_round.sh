set -u
python -m pytest tests/test_gpu_forecast.py tests/test_gpu_iewpf.py -q -x > gpurun_out/t.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/t.log
for v in base new base new; do
  echo -n "$v "; DC_LIB_PATH=$PWD/variants/$v.so python bench.py --no-cpu-baseline --steps 10 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['ms_per_step'], d['value'])"
done
export DC_NO_GRAPH=1
for v in base new; do
  DC_LIB_PATH=$PWD/variants/$v.so python tools/profile_cycle.py --cycles 1 > /dev/null 2>&1 && \
  DC_LIB_PATH=$PWD/variants/$v.so ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/l_$v.csv python tools/profile_cycle.py --cycles 1 > /dev/null 2>&1
  echo "$v ncu rc=$?"
done
