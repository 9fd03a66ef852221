set -u
O=gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/r2m_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 $O/r2m_pytest.log
python bench.py --nx 500 --ny 300 --members-total 100 --no-cpu-baseline --steps 20 --warmup 3 > $O/r2m_c1.json 2>$O/r2m_c1.err; echo "c1 rc=$?"
python bench.py --nx 500 --ny 300 --members-total 100 --obs moorings --no-cpu-baseline --steps 20 --warmup 3 > $O/r2m_c2.json 2>$O/r2m_c2.err; echo "c2 rc=$?"
