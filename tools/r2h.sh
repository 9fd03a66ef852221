set -u
O=gpurun_out
python bench.py --nx 500 --ny 300 --members-total 100 --no-cpu-baseline --steps 20 --warmup 3 > $O/r2h_c1.json 2>$O/r2h_c1.err; echo "c1 rc=$?"
python bench.py --nx 500 --ny 300 --members-total 100 --obs moorings --no-cpu-baseline --steps 20 --warmup 3 > $O/r2h_c2.json 2>$O/r2h_c2.err; echo "c2 rc=$?"
