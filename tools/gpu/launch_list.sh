#!/bin/bash
# ncu launch list (gpu__time_duration only) of the repo kernels of one matvec: WL=cfg3 tools/gpu/launch_list.sh
set -u
cd ${GRAFT_REPO_ROOT:-.}
OUT=gpurun_out/launches; mkdir -p $OUT
NCU=/usr/local/cuda/bin/ncu
export DEFMM_PLAN_BUILD=host
for w in ${WL:-cfg2_l6 cfg3}; do
  B="python bench.py --workload $w ${DT:+--dtype $DT} --steps 1 --warmup 0 --no-cpu-baseline --no-secondary --profile"
  timeout 600 $B > $OUT/plain_$w.log 2>&1 && \
  timeout 1500 $NCU --metrics gpu__time_duration.sum --clock-control none -k regex:'p2m|m2m|m2f|m2l|f2l|l2l|l2p|p2p' \
     --csv --log-file $OUT/launches_$w${DT:+_$DT}.csv $B > $OUT/ncu_$w.log 2>&1
  python - <<P
import csv, collections
rows = list(csv.reader(open("$OUT/launches_$w${DT:+_$DT}.csv", errors="ignore")))
h = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
hd = rows[h]; ki, vi = hd.index("Kernel Name"), hd.index("Metric Value")
acc = collections.OrderedDict()
for r in rows[h + 1:]:
    if len(r) > vi:
        k = r[ki].split("(")[0][-40:]
        a = acc.setdefault(k, [0, 0.0]); a[0] += 1; a[1] += float(r[vi].replace(",", "")) / 1e3
print("$w ${DT:-}")
for k, (n, t) in acc.items():
    print(f"  {t:10.1f} us  x{n:3d}  {k}")
P
done
