#!/bin/bash
# The repo's memory checker over the whole GPU suite (compute-sanitizer is closed on the
# GPU pool): every device buffer guard-banded and poisoned (DC_GUARD=1, csrc/guard.cu);
# tests/conftest.py verifies every guard band after each GPU test; the bitwise oracle
# comparisons catch poisoned (uninitialised / out-of-bounds) reads. Graph path and the
# host-driven substep loop. Usage (under gpurun): bash tools/guardcheck.sh [tag]
set -u
TAG=${1:-r2}
O=gpurun_out
mkdir -p $O
DC_GUARD=1 timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/guardcheck_${TAG}_graph.log 2>&1
echo "guard graph rc=$? $(tail -1 $O/guardcheck_${TAG}_graph.log)"
DC_GUARD=1 DC_NO_GRAPH=1 timeout 2400 python -m pytest tests/test_gpu_forecast.py tests/test_gpu_iewpf.py tests/test_gpu_configs.py -m gpu -q -p no:cacheprovider -k "not configs0 and not configs4" > $O/guardcheck_${TAG}_hostloop.log 2>&1
echo "guard hostloop rc=$? $(tail -1 $O/guardcheck_${TAG}_hostloop.log)"
