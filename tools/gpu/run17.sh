cd $GRAFT_REPO_ROOT
O=gpurun_out/r17; mkdir -p $O
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $O/smoke.log 2>&1
timeout 1800 python -m pytest tests -m gpu -q -x > $O/tests.log 2>&1
echo "tests rc=$?" >> $O/rc.txt
timeout 1500 python tools/gpu/time_build.py cfg2 cfg3 cfg5 cfg4 > $O/time_build.log 2>&1
