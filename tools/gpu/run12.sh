cd $GRAFT_REPO_ROOT
O=gpurun_out/r12; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_operators.py -m gpu -q > $O/tests_ops.log 2>&1
echo "ops rc=$?" >> $O/rc.txt
timeout 900 python tools/gpu/c64_bar.py > $O/c64_bar.log 2>&1
timeout 600 python tools/sanitize_case.py > $O/allmodes.log 2>&1
echo "allmodes rc=$?" >> $O/rc.txt
