set -u
echo -n "u2 bitwise: "; DC_LIB_PATH=$PWD/variants/u2.so timeout 120 python tools/tiny_step.py 500 300 3 2>&1 | tail -1
echo -n "u2 bitwise small: "; DC_LIB_PATH=$PWD/variants/u2.so timeout 120 python tools/tiny_step.py 100 60 2 2>&1 | tail -1
bash tools/ab_forecast.sh cur u2 2>&1
