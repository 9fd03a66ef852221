set -u
timeout 900 python -m pytest tests/test_gpu_forecast.py -m gpu -q -p no:cacheprovider -k "many_members or bitwise_10 or launch_variants or shapes or flux_rhs" 2>&1 | tail -2
bash tools/ab_forecast.sh g2 cur 2>&1
