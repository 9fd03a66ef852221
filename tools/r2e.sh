set -u
echo -n "s1b4 bitwise: "; DC_LIB_PATH=$PWD/variants/s1b4.so timeout 120 python tools/tiny_step.py 500 300 3 2>&1 | tail -1
bash tools/ab_forecast.sh cur s1b4 2>&1
