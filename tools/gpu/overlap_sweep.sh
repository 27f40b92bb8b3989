#!/bin/bash
# P2P placement sweep: bench lines for each workload x (overlap, far-priority)
mkdir -p gpurun_out/ovl
for w in ${WORKLOADS:-cfg3 cfg5 cfg2_l6 cfg4}; do
  for v in "upward 0" "m2l 1" "m2l 0" "m2m 0"; do
    set -- $v
    python bench.py --workload $w --steps 5 --warmup 3 --no-secondary --no-cpu-baseline \
      --p2p-overlap $1 --far-priority $2 > gpurun_out/ovl/${w}_$1_$2.json 2> gpurun_out/ovl/${w}_$1_$2.err
    python - <<P
import json
try:
    d = json.loads(open("gpurun_out/ovl/${w}_$1_$2.json").read().strip().splitlines()[-1])
    print("$w", "$1", "$2", round(d["ms_per_step"], 3), {k: round(v, 2) for k, v in d.get("stages_ms", {}).items()})
except Exception as e:
    print("$w $1 $2 failed", e)
P
  done
done
