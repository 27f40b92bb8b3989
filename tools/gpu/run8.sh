cd $GRAFT_REPO_ROOT
O=gpurun_out/r8; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
for rep in 1 2; do
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --m2l-levels staged > $O/bench_cfg2_staged_b3_$rep.log 2>&1
done
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > $O/bench_cfg2_auto.log 2>&1
DEFMM_NVCC_FLAGS=-DDEFMM_STAGE_MINB=2 python -m paper_2202_04894_b200.build --force > $O/build2.log 2>&1
DEFMM_STAGE_SLOTS=64 timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --m2l-levels staged > $O/bench_cfg2_staged_b2_ns64.log 2>&1
