set -u
O=gpurun_out
timeout 1200 python -m pytest tests/test_gpu_forecast.py tests/test_gpu_iewpf.py -m gpu -q -p no:cacheprovider > $O/r2n_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 $O/r2n_pytest.log
bash tools/ab_forecast.sh cur 2>&1
