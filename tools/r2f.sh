set -u
O=gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/r2f_pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 $O/r2f_pytest_gpu.log
bash tools/guardcheck.sh r2f
timeout 900 python bench.py --no-cpu-baseline > $O/r2f_bench.json 2> $O/r2f_bench.err; echo "bench rc=$?"; tail -3 $O/r2f_bench.err
