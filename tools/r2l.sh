set -u
for rep in 1 2; do for v in cur nobox; do
  if [ $v = cur ]; then L=""; else L=$PWD/variants/$v.so; fi
  echo -n "$v c2: "; DC_LIB_PATH=$L python bench.py --nx 500 --ny 300 --members-total 100 --obs moorings --no-cpu-baseline --steps 20 --warmup 3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d['cycle_ms'],3), [ (k['kernel'], round(k['us_per_launch'],1)) for k in d['roofline']['kernels'] if k['kernel'] in ('pull_apply','pull_tables')])"
done; done
