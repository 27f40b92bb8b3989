# staged M2L (K7 v13): parity + timing; P2P persistent-grid overlap sweep on cfg5
cd $GRAFT_REPO_ROOT
O=gpurun_out/r3; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "canonical_gather or group_m2l" > $O/tests_staged.log 2>&1
echo "tests rc=$?" >> $O/rc.txt
for ns in 48 32 64; do
  DEFMM_STAGE_SLOTS=$ns timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --m2l-levels staged > $O/bench_cfg2_staged_ns$ns.log 2>&1
  echo "bench ns=$ns rc=$?" >> $O/rc.txt
done
for g in 148 296 444; do for fp in 0 1; do
  timeout 600 python bench.py --workload cfg5 --steps 5 --warmup 3 --no-cpu-baseline --no-secondary --p2p-overlap m2l --p2p-grid $g --far-priority $fp > $O/cfg5_m2l_grid${g}_fp$fp.log 2>&1
done; done
