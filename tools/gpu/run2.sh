# baseline validation + overlap sweep (round 2, re-entry)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r2
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r2/smoke.log 2>&1
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/r2/tests.log 2>&1
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2/bench_cfg2.log 2>&1
for ov in upward m2l; do for fp in 0 1; do
  timeout 600 python bench.py --workload cfg5 --steps 5 --warmup 3 --no-cpu-baseline --no-secondary --p2p-overlap $ov --far-priority $fp > gpurun_out/r2/cfg5_${ov}_fp$fp.log 2>&1
  timeout 600 python bench.py --workload cfg3 --steps 5 --warmup 3 --no-cpu-baseline --no-secondary --p2p-overlap $ov --far-priority $fp > gpurun_out/r2/cfg3_${ov}_fp$fp.log 2>&1
done; done
