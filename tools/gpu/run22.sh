cd $GRAFT_REPO_ROOT
O=gpurun_out/r22; mkdir -p $O
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $O/smoke.log 2>&1
timeout 1800 python -m pytest tests -m gpu -q > $O/tests.log 2>&1
echo "tests rc=$?" >> $O/rc.txt
timeout 900 python bench.py --workload cfg3 --steps 5 --warmup 3 --no-cpu-baseline > $O/bench_cfg3.log 2>&1
timeout 900 python bench.py --workload cfg2_l6 --steps 5 --warmup 3 --no-cpu-baseline > $O/bench_cfg2_l6.log 2>&1
timeout 900 python bench.py > $O/bench_default.log 2>&1
SPECS_SKIP=1 bash tools/gpu/prof_r02.sh > $O/prof.log 2>&1
