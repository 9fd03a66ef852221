set -u
O=gpurun_out
timeout 600 python -m pytest tests/test_gpu_experiment.py tests/test_gpu_cpp_driver.py -q -x > $O/r2c_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 $O/r2c_pytest.log
export DC_NO_GRAPH=1
timeout 300 python tools/profile_cycle.py --nx 1000 --ny 600 --members 125 --cycles 1 > $O/r2c_pc.log 2>&1; echo "pc rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:swe_stage_pair -c 2 -o $O/full_swe_r2c -f python tools/profile_cycle.py --nx 1000 --ny 600 --members 125 --cycles 1 > $O/r2c_ncu_swe.log 2>&1; echo "ncu swe rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_r2c.csv python tools/profile_cycle.py --nx 1000 --ny 600 --members 125 --cycles 1 > $O/r2c_ncu_launch.log 2>&1; echo "launch list rc=$?"
