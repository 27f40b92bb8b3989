cd $GRAFT_REPO_ROOT
O=gpurun_out/r16; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_build.py -m gpu -q -x > $O/tests.log 2>&1
echo "tests rc=$?" >> $O/rc.txt
