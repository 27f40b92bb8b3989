#!/bin/bash
# Round-2 profiling pass (run under gpurun, one GPU):
#  1. per-launch metrics of one cfg2 matvec (c64 and c128): time, DRAM bytes,
#     L2->L1 bytes, FP32/FP64/XU pipe utilisation -> profiles/r02_m2l_ncu.json,
#     profiles/r02_p2p_pipes.json (tools/summarise_ncu_r02.py)
#  2. ncu --set full of the dominant kernels: the c64 quartet and c128 staged M2L (cfg2), the
#     cfg5 blocked M2L, the mutual P2P in both precisions
set -u
cd ${GRAFT_REPO_ROOT:-.}
# the plan is built by the host builders here: under ncu every torch sort/scan of the device
# builders would be profiled too (same trees and lists either way)
export DEFMM_PLAN_BUILD=host
OUT=gpurun_out/prof_r02; mkdir -p $OUT
NCU=/usr/local/cuda/bin/ncu
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,l1tex__m_xbar2l1tex_read_bytes.sum,lts__t_sectors_srcunit_tex_op_read.sum,sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active,sm__inst_issued.avg.pct_of_peak_sustained_active,lts__throughput.avg.pct_of_peak_sustained_elapsed,l1tex__throughput.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active
for DT in ${METRIC_DTYPES-c64 c128}; do
  B="python bench.py --workload cfg2 --dtype $DT --steps 1 --warmup 0 --no-cpu-baseline --no-secondary --profile"
  timeout 600 $B > $OUT/plain_$DT.log 2>&1 && \
  timeout 900 $NCU --metrics $M --clock-control none --csv --log-file $OUT/metrics_cfg2_$DT.csv $B > $OUT/ncu_$DT.log 2>&1
  echo "metrics $DT rc=$?" >> $OUT/rc.txt
done
[ -n "${SPECS_SKIP:-}" ] && exit 0
for spec in "cfg2 c64 m2l_group" "cfg2 c128 m2l_stage" "cfg5 c128 m2l_blocked" "cfg5 c128 p2p_mut_kernel" "cfg2 c64 p2p_mut_f32"; do
  set -- $spec
  B="python bench.py --workload $1 --dtype $2 --steps 1 --warmup 0 --no-cpu-baseline --no-secondary --profile"
  timeout 600 $B > $OUT/plain_$1_$3.log 2>&1 && \
  timeout 1200 $NCU --set full --clock-control none --import-source on -k regex:$3 -s 0 -c 1 -o $OUT/full_$1_$2_$3 -f $B > $OUT/full_$1_$3.log 2>&1
  echo "full $1 $3 rc=$?" >> $OUT/rc.txt
  $NCU -i $OUT/full_$1_$2_$3.ncu-rep --page raw --csv > $OUT/full_$1_$2_$3.raw.csv 2>/dev/null
  $NCU -i $OUT/full_$1_$2_$3.ncu-rep --page details --csv > $OUT/full_$1_$2_$3.details.csv 2>/dev/null
  $NCU -i $OUT/full_$1_$2_$3.ncu-rep --page source --csv > $OUT/full_$1_$2_$3.source.csv 2>/dev/null
  rm -f $OUT/full_$1_$2_$3.ncu-rep
done
