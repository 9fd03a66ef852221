set -u
O=gpurun_out
timeout 1800 python -m pytest tests -m gpu -q > $O/r2b_pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -15 $O/r2b_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/r2b_smoke.log 2>&1; echo "smoke rc=$?"; tail -2 $O/r2b_smoke.log
timeout 900 python bench.py > $O/r2b_bench.json 2> $O/r2b_bench.err; echo "bench rc=$?"; tail -c 3000 $O/r2b_bench.json; tail -5 $O/r2b_bench.err
