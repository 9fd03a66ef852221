set -u
O=gpurun_out
timeout 1200 python -m pytest tests/test_gpu_iewpf.py tests/test_gpu_configs.py tests/test_gpu_experiment.py tests/test_gpu_bench_ranks.py -m gpu -q -x -p no:cacheprovider > $O/r2i_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 $O/r2i_pytest.log
python bench.py --nx 500 --ny 300 --members-total 100 --obs moorings --no-cpu-baseline --steps 20 --warmup 3 > $O/r2i_c2.json 2>$O/r2i_c2.err; echo "c2 rc=$?"
python bench.py --nx 500 --ny 300 --members-total 100 --no-cpu-baseline --steps 20 --warmup 3 > $O/r2i_c1.json 2>$O/r2i_c1.err; echo "c1 rc=$?"
export DC_NO_GRAPH=1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:pull_apply -c 1 -o $O/full_pull_r2i -f python tools/profile_cycle.py --obs moorings --cycles 1 > $O/r2i_ncu.log 2>&1; echo "ncu rc=$?"
