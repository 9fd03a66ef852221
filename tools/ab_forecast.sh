#!/bin/bash
# A/B model-step throughput of library variants (variants/NAME.so or "cur" = the in-tree
# build), interleaved twice, at 500x300 x 100 members and 1000x600 x 250 members.
# Usage: tools/ab_forecast.sh NAME [NAME ...]
for rep in 1 2; do for v in "$@"; do
  if [ "$v" = cur ]; then lib=""; else lib=$PWD/variants/$v.so; fi
  for sz in "--nx 500 --ny 300 --members 100" "--nx 1000 --ny 600 --members 250"; do
    echo -n "$v [$sz] "
    DC_LIB_PATH=$lib timeout 300 python tools/quick_forecast_bench.py $sz --steps 10 2>&1 | grep -E "ms/model-step|Error|error" | head -2
  done
done; done
