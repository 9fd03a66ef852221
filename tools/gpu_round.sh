#!/bin/bash
# One GPU session: tests, bench line, launch list and ncu --set full captures of the top
# kernels (each ncu pass only after the same command exited 0 without ncu).
# Usage (under gpurun): bash tools/gpu_round.sh [tag]
set -u
TAG=${1:-r1}
O=gpurun_out
mkdir -p $O
python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 $O/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"
python bench.py > $O/bench.json 2> $O/bench.err; echo "bench rc=$?"; tail -c 600 $O/bench.json
python bench.py --obs moorings --no-cpu-baseline > $O/bench_moorings.json 2> $O/bench_moorings.err; echo "moorings rc=$?"
python bench.py --impl reference --steps 3 --warmup 1 > $O/bench_ref.json 2> $O/bench_ref.err; echo "ref rc=$?"
python bench.py --nx 1000 --ny 600 --members 125 --steps 5 --warmup 3 --no-cpu-baseline > $O/bench_configs4.json 2> $O/bench_configs4.err; echo "configs4 rc=$?"
python tools/e2e_probe.py --cycles 10 > $O/e2e_probe.log 2>&1; echo "e2e probe rc=$?"
export DC_NO_GRAPH=1
if python tools/profile_cycle.py --cycles 2 > $O/profile_cycle.log 2>&1; then
  ncu --metrics gpu__time_duration.sum --clock-control none --csv \
      --log-file $O/launches_${TAG}.csv python tools/profile_cycle.py --cycles 2 > $O/ncu_launch.log 2>&1
  echo "launch list rc=$?"
  ncu --set full --clock-control none --import-source on -k regex:swe_stage_pair -c 2 \
      -o $O/full_swe_${TAG} -f python tools/profile_cycle.py --cycles 1 > $O/ncu_full_swe.log 2>&1
  echo "ncu full swe rc=$?"
  for k in q_half_apply pull_apply local_blocks philox_soar; do
    ncu --set full --clock-control none --import-source on -k regex:$k -c 1 \
        -o $O/full_${k}_${TAG} -f python tools/profile_cycle.py --cycles 1 > $O/ncu_full_$k.log 2>&1
    echo "ncu full $k rc=$?"
  done
fi
