cd $GRAFT_REPO_ROOT
O=gpurun_out/r5; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "canonical_gather or group_m2l" > $O/tests_staged.log 2>&1
echo "tests rc=$?" >> $O/rc.txt
run() { # tag ns depth
  DEFMM_STAGE_SLOTS=$2 DEFMM_STAGE_DEPTH=$3 timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --m2l-levels staged > $O/bench_cfg2_$1_ns$2_d$3.log 2>&1
  echo "bench $1 ns=$2 d=$3 rc=$?" >> $O/rc.txt
}
run b3 48 3; run b3 32 4; run b3 24 6; run b3 72 2
DEFMM_NVCC_FLAGS=-DDEFMM_STAGE_MINB=2 python -m paper_2202_04894_b200.build --force > $O/build2.log 2>&1
run b2 48 3; run b2 64 3; run b2 48 4; run b2 96 2
