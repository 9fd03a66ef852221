set -u
O=gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1200 python -m pytest tests -m gpu -q -x > $O/r2a_pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -5 $O/r2a_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/r2a_smoke.log 2>&1; echo "smoke rc=$?"; tail -2 $O/r2a_smoke.log
timeout 600 python bench.py > $O/r2a_bench.json 2> $O/r2a_bench.err; echo "bench rc=$?"; tail -c 1500 $O/r2a_bench.json
timeout 900 python bench.py --nx 1000 --ny 600 --members 1000 --steps 5 --warmup 3 --no-cpu-baseline > $O/r2a_bench_c4.json 2> $O/r2a_bench_c4.err; echo "configs4 rc=$?"; tail -c 800 $O/r2a_bench_c4.json; tail -5 $O/r2a_bench_c4.err
