# A/B bench.py cycle time under environment settings: each arg is "NAME:VAR=VAL,VAR=VAL"
for rep in 1 2; do for v in "$@"; do
  name=${v%%:*}; envs=${v#*:}
  echo -n "$name "; env $(echo $envs | tr ',' ' ') python bench.py --no-cpu-baseline --steps 10 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('ms/cycle %.3f' % d['ms_per_step'], 'value %.4g' % d['value'], 'e2e %.3f' % d['e2e']['ms_per_step'])"
done; done
