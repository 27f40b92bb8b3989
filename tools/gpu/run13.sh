cd $GRAFT_REPO_ROOT
O=gpurun_out/r13; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "canonical_gather or group_m2l" > $O/tests.log 2>&1
echo "tests rc=$?" >> $O/rc.txt
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --m2l-levels cousins > $O/bench_cfg2_cousins.log 2>&1
DEFMM_NVCC_FLAGS="-DDEFMM_COUSIN_MINB=2" python -m paper_2202_04894_b200.build --force > $O/build2.log 2>&1
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --m2l-levels cousins > $O/bench_cfg2_cousins_minb2.log 2>&1
