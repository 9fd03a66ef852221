# A/B bench.py cycle time of library variants (variants/*.so), interleaved twice.
for v in "$@" "$@"; do
  echo -n "$v "; DC_LIB_PATH=$PWD/variants/$v.so python bench.py --no-cpu-baseline --steps 10 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('ms/cycle %.3f' % d['ms_per_step'], 'value %.4g' % d['value'], 'launches', d['gpu_launches'])"
done
