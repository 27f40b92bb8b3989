cd $GRAFT_REPO_ROOT
O=gpurun_out/r20; mkdir -p $O
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $O/smoke.log 2>&1
timeout 1800 python -m pytest tests -m gpu -q -x > $O/tests.log 2>&1
echo "tests rc=$?" >> $O/rc.txt
for ov in upward m2l; do for fp in 0 1; do
  timeout 600 python bench.py --dtype c128 --steps 10 --warmup 3 --no-cpu-baseline --no-secondary --p2p-overlap $ov --far-priority $fp > $O/cfg2_c128_${ov}_fp$fp.log 2>&1
done; done
timeout 600 python bench.py --workload cfg1 --steps 10 --warmup 3 --no-cpu-baseline > $O/bench_cfg1.log 2>&1
timeout 600 python bench.py --workload cfg5 --steps 5 --warmup 3 --no-cpu-baseline --no-secondary > $O/bench_cfg5.log 2>&1
