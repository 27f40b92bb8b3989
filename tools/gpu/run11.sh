cd $GRAFT_REPO_ROOT
O=gpurun_out/r11; mkdir -p $O
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $O/smoke.log 2>&1
timeout 1800 python -m pytest tests -m gpu -q -x > $O/tests.log 2>&1
echo "tests rc=$?" >> $O/rc.txt
for w in cfg2 cfg5 cfg3; do
  timeout 600 python bench.py --workload $w --steps 5 --warmup 3 --no-cpu-baseline > $O/bench_${w}_mut.log 2>&1
done
DEFMM_NVCC_FLAGS="-DDEFMM_P2P_MUT_MINB64=3" python -m paper_2202_04894_b200.build --force > $O/build2.log 2>&1
timeout 600 python bench.py --workload cfg5 --steps 5 --warmup 3 --no-cpu-baseline --no-secondary > $O/bench_cfg5_mut_minb3.log 2>&1
