cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r1_smoke.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r1_tests.log 2>&1
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/r1_bench.log 2>&1
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r1_ref.log 2>&1
nproc > gpurun_out/r1_nproc.txt
