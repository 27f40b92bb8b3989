cd $GRAFT_REPO_ROOT
O=gpurun_out/r14; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
for ov in upward m2l full m2m; do for fp in 0 1; do
  timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-secondary --p2p-overlap $ov --far-priority $fp > $O/cfg2_${ov}_fp$fp.log 2>&1
done; done
