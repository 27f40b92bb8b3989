#!/bin/bash
# Round-2 final measurement pass: GPU tests, every BASELINE workload, the reference arm,
# ncu launch metrics + full captures of the current dominant kernels.
set -u
cd ${GRAFT_REPO_ROOT:-.}
O=gpurun_out/final; mkdir -p $O
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $O/smoke.log 2>&1
timeout 1800 python -m pytest tests -m gpu -q > $O/tests.log 2>&1
echo "tests rc=$?" >> $O/rc.txt
timeout 900 python bench.py > $O/bench_default.log 2>&1
echo "bench rc=$?" >> $O/rc.txt
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > $O/bench_reference.log 2>&1
for w in cfg1 cfg2_l6 cfg3 cfg5 cfg5_l6 cfg5_l8 cfg4; do
  timeout 1200 python bench.py --workload $w --steps 5 --warmup 3 --no-cpu-baseline > $O/bench_$w.log 2>&1
done
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --m2l-levels staged > $O/bench_cfg2_staged.log 2>&1
