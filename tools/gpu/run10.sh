cd $GRAFT_REPO_ROOT
O=gpurun_out/r10; mkdir -p $O
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $O/smoke.log 2>&1
timeout 1800 python -m pytest tests -m gpu -q -x > $O/tests.log 2>&1
echo "tests rc=$?" >> $O/rc.txt
for w in cfg2 cfg5 cfg3; do
  for g in 0 1184; do
    timeout 600 python bench.py --workload $w --steps 5 --warmup 3 --no-cpu-baseline --p2p-grid $g > $O/bench_${w}_mut_g$g.log 2>&1
  done
  DEFMM_P2P_MUTUAL=0 timeout 600 python bench.py --workload $w --steps 5 --warmup 3 --no-cpu-baseline > $O/bench_${w}_old.log 2>&1
done
