#!/bin/bash
# Profiling pass for one workload on the GPU box (run under gpurun):
#   tools/profile_gpu.sh <workload> <tag> [extra bench args]
# 1. launch list of one eager matvec (times + DRAM bytes per launch, cold cache)
# 2. one `ncu --set full` capture of the top M2L kernel and of the P2P kernel
# Outputs under gpurun_out/prof_<tag>/ (summarised into profiles/ afterwards).
set -u
W=$1; TAG=$2; shift 2
OUT=gpurun_out/prof_$TAG; mkdir -p $OUT
B="python bench.py --workload $W --steps 1 --warmup 3 --no-cpu-baseline --no-secondary --profile $*"
NCU=/usr/local/cuda/bin/ncu
timeout 600 $NCU --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    --csv --log-file $OUT/launches.csv $B > $OUT/launches.log 2>&1
echo "launches rc=$?" >> $OUT/rc.txt
for K in ${KERNELS:-m2l_rows_kernel p2p}; do
  timeout 900 $NCU --set full --clock-control none --import-source on -k regex:$K -s 0 -c 1 \
      -o $OUT/full_$K -f $B > $OUT/full_$K.log 2>&1
  echo "full $K rc=$?" >> $OUT/rc.txt
  $NCU -i $OUT/full_$K.ncu-rep --page raw --csv > $OUT/full_$K.raw.csv 2>/dev/null
  $NCU -i $OUT/full_$K.ncu-rep --page details --csv > $OUT/full_$K.details.csv 2>/dev/null
  $NCU -i $OUT/full_$K.ncu-rep --page source --csv > $OUT/full_$K.source.csv 2>/dev/null
  # the .ncu-rep files would exceed gpurun's 64 MiB return limit
  [ "${KEEP_REP:-0}" = 1 ] || rm -f $OUT/full_$K.ncu-rep
done
