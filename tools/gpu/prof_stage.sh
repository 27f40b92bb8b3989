#!/bin/bash
# ncu --set full of the staged M2L kernel on cfg2 (c64), after a plain run exits 0
set -u
cd ${GRAFT_REPO_ROOT:-.}
OUT=gpurun_out/prof_stage; mkdir -p $OUT
NCU=/usr/local/cuda/bin/ncu
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
B="python bench.py --workload ${WL:-cfg2} --dtype ${DT:-c64} --steps 1 --warmup 0 --no-cpu-baseline --no-secondary --profile --m2l-levels ${MODE:-staged}"
timeout 600 $B > $OUT/plain.log 2>&1 && \
timeout 1200 $NCU --set full --clock-control none --import-source on -k regex:${KERN:-m2l_stage} -s 0 -c 1 -o $OUT/full -f $B > $OUT/ncu.log 2>&1
echo "rc=$?" > $OUT/rc.txt
$NCU -i $OUT/full.ncu-rep --page raw --csv > $OUT/full.raw.csv 2>/dev/null
$NCU -i $OUT/full.ncu-rep --page details --csv > $OUT/full.details.csv 2>/dev/null
$NCU -i $OUT/full.ncu-rep --page source --csv > $OUT/full.source.csv 2>/dev/null
rm -f $OUT/full.ncu-rep
