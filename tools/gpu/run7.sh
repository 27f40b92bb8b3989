cd $GRAFT_REPO_ROOT
O=gpurun_out/r7; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "canonical_gather or group_m2l" > $O/tests_staged.log 2>&1
echo "tests rc=$?" >> $O/rc.txt
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --m2l-levels staged > $O/bench_cfg2_staged.log 2>&1
timeout 600 python bench.py --workload cfg3 --steps 5 --warmup 3 --no-cpu-baseline --m2l-levels staged > $O/bench_cfg3_staged.log 2>&1
timeout 600 python bench.py --workload cfg3 --steps 5 --warmup 3 --no-cpu-baseline > $O/bench_cfg3_auto.log 2>&1
timeout 900 python bench.py --workload cfg5 --steps 5 --warmup 3 --no-cpu-baseline --no-secondary --m2l-levels staged_all > $O/bench_cfg5_staged_all.log 2>&1
