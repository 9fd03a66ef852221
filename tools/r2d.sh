set -u
O=gpurun_out
for v in o0 o1 o2b4; do echo -n "$v bitwise: "; DC_LIB_PATH=$PWD/variants/$v.so timeout 120 python tools/tiny_step.py 500 300 3 2>&1 | tail -1; done
echo -n "cur bitwise: "; timeout 120 python tools/tiny_step.py 500 300 3 2>&1 | tail -1
bash tools/ab_forecast.sh o0 cur o1 o2b4 2>&1
