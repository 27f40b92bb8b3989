cd $GRAFT_REPO_ROOT
O=gpurun_out/r21; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 900 python bench.py --workload cfg2_l6 --steps 5 --warmup 3 --no-cpu-baseline --m2l-levels staged > $O/bench_cfg2_l6_staged.log 2>&1
timeout 900 python bench.py --workload cfg3 --steps 5 --warmup 3 --no-cpu-baseline --m2l-levels staged > $O/bench_cfg3_staged.log 2>&1
timeout 1200 python bench.py --workload cfg4 --steps 3 --warmup 3 --no-cpu-baseline --no-secondary --m2l-levels staged > $O/bench_cfg4_staged.log 2>&1
timeout 900 python bench.py --workload cfg5 --steps 5 --warmup 3 --no-cpu-baseline --no-secondary --m2l-levels staged_all > $O/bench_cfg5_staged_all.log 2>&1
