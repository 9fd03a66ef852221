#!/bin/bash
# compute-sanitizer over the GPU suite's small cases: memcheck (out-of-bounds
# / misaligned accesses, leaks), racecheck (shared-memory hazards), synccheck (barrier and
# mbarrier misuse), with the graph path and the host-driven loop (DC_NO_GRAPH=1).
# Usage (under gpurun): bash tools/sanitize.sh [tag]
set -u
TAG=${1:-r2}
O=gpurun_out
mkdir -p $O
CS="compute-sanitizer --target-processes all --error-exitcode 86 --print-limit 20"
SMALL="tests/test_gpu_forecast.py tests/test_gpu_iewpf.py tests/test_gpu_experiment.py"
DESEL="not exhaustive and not fma_tolerance and not shapes and not full_size and not refined and not count_edges and not twenty and not generate_truth and not snapshot_bytes"
run() {  # name env tool extra-pytest-args
  local name=$1 env=$2 tool=$3; shift 3
  env $env timeout 3000 $CS --tool $tool python -m pytest -q -x -p no:cacheprovider "$@" \
    > $O/sanitizer_${TAG}_${name}.log 2>&1
  echo "$name rc=$? $(grep -E 'ERROR SUMMARY|passed|failed' $O/sanitizer_${TAG}_${name}.log | tail -2 | tr '\n' ' ')"
}
run memcheck_graph "DC_X=0" memcheck $SMALL -m gpu -k "$DESEL"
run memcheck_hostloop "DC_NO_GRAPH=1" memcheck tests/test_gpu_forecast.py tests/test_gpu_iewpf.py -m gpu -k "$DESEL"
run racecheck "DC_NO_GRAPH=1" racecheck tests/test_gpu_forecast.py tests/test_gpu_iewpf.py -m gpu -k "bitwise_10_members or launch_variants or assimilate_bitwise and 100 or da_cycle_matches or two_slices"
run synccheck "DC_NO_GRAPH=1" synccheck tests/test_gpu_forecast.py tests/test_gpu_iewpf.py -m gpu -k "bitwise_10_members or launch_variants or assimilate_bitwise and 100 or da_cycle_matches or two_slices"
run initcheck "DC_NO_GRAPH=1" initcheck tests/test_gpu_iewpf.py -m gpu -k "da_cycle_matches or assimilate_bitwise and 100"
