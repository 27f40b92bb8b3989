cd $GRAFT_REPO_ROOT
O=gpurun_out/r4; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
for ns in 48 32 64; do
  DEFMM_STAGE_SLOTS=$ns timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --m2l-levels staged > $O/bench_cfg2_staged_ns$ns.log 2>&1
  echo "bench ns=$ns rc=$?" >> $O/rc.txt
done
timeout 600 python bench.py --workload cfg3 --steps 5 --warmup 3 --no-cpu-baseline --no-secondary --m2l-levels staged > $O/bench_cfg3_staged.log 2>&1
timeout 600 python bench.py --workload cfg5 --steps 5 --warmup 3 --no-cpu-baseline --no-secondary --m2l-levels staged_all > $O/bench_cfg5_staged_all.log 2>&1
