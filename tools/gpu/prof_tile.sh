cd $GRAFT_REPO_ROOT
export DEFMM_TILE_Q=4 DEFMM_TILE_K=4 DEFMM_TILE_OPS=768 DEFMM_TILE_EV=2048
NCU=/usr/local/cuda/bin/ncu
OUT=gpurun_out/pt; mkdir -p $OUT
timeout 900 $NCU --set full --clock-control none --import-source on -k regex:m2l_tile -s 0 -c 1 -o $OUT/tile -f \
   python bench.py --workload cfg2 --steps 1 --warmup 1 --no-cpu-baseline --no-secondary --profile --m2l-levels tiles > $OUT/ncu.log 2>&1
$NCU -i $OUT/tile.ncu-rep --page raw --csv > $OUT/tile.raw.csv 2>/dev/null
$NCU -i $OUT/tile.ncu-rep --page details --csv > $OUT/tile.details.csv 2>/dev/null
$NCU -i $OUT/tile.ncu-rep --page source --csv > $OUT/tile.source.csv 2>/dev/null
rm -f $OUT/tile.ncu-rep
