#!/bin/bash
# End-of-round evidence on one GPU (under gpurun): GPU suite, smoke, the default bench line,
# the reference arm on the same config, the library communicator path at N=1, and the ncu
# launch list + full capture of the stage kernels (each ncu pass only after the same command
# exited 0 without ncu). Usage: bash tools/final_round.sh TAG
set -u
TAG=${1:-r2}
O=gpurun_out
mkdir -p $O
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/${TAG}_pytest_gpu.log 2>&1; echo "pytest rc=$? $(tail -1 $O/${TAG}_pytest_gpu.log)"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/${TAG}_smoke.log 2>&1; echo "smoke rc=$? $(tail -1 $O/${TAG}_smoke.log)"
timeout 900 python bench.py --steps 20 --warmup 5 > $O/${TAG}_bench.json 2> $O/${TAG}_bench.err; echo "bench rc=$?"
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > $O/${TAG}_bench_ref.json 2> $O/${TAG}_bench_ref.err; echo "ref rc=$?"
timeout 600 python bench.py --nx 500 --ny 300 --members-total 100 --no-cpu-baseline --comm > $O/${TAG}_bench_comm_c1.json 2> $O/${TAG}_bench_comm_c1.err; echo "comm c1 rc=$?"
timeout 600 python bench.py --nx 500 --ny 300 --members-total 100 --no-cpu-baseline > $O/${TAG}_bench_c1.json 2> $O/${TAG}_bench_c1.err; echo "c1 rc=$?"
timeout 600 python bench.py --nx 500 --ny 300 --members-total 100 --obs moorings --no-cpu-baseline > $O/${TAG}_bench_c2.json 2> $O/${TAG}_bench_c2.err; echo "c2 rc=$?"
export DC_NO_GRAPH=1
if timeout 300 python tools/profile_cycle.py --nx 1000 --ny 600 --members 125 --cycles 1 > $O/${TAG}_pc.log 2>&1; then
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/${TAG}_launches.csv python tools/profile_cycle.py --nx 1000 --ny 600 --members 125 --cycles 1 > $O/${TAG}_ncu_launch.log 2>&1; echo "launch list rc=$?"
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:swe_stage_pair -c 2 -o $O/${TAG}_full_swe -f python tools/profile_cycle.py --nx 1000 --ny 600 --members 125 --cycles 1 > $O/${TAG}_ncu_swe.log 2>&1; echo "ncu swe rc=$?"
  for k in q_half_apply pull_apply; do
    timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -c 1 -o $O/${TAG}_full_$k -f python tools/profile_cycle.py --nx 1000 --ny 600 --members 125 --cycles 1 > $O/${TAG}_ncu_$k.log 2>&1; echo "ncu $k rc=$?"
  done
fi
