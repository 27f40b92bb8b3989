# M2L sliced-tile sweep on cfg2 (isolated M2L stage time per configuration)
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "canonical or group_m2l" > gpurun_out/st_tests.log 2>&1
B="python bench.py --steps 5 --warmup 2 --no-cpu-baseline --no-secondary"
timeout 300 $B > gpurun_out/st_auto.log 2>&1
for Q in 8; do for K in 4; do for OPS in 2048 4096; do for EV in 4096 16384; do
  DEFMM_TILE_L1=1 DEFMM_TILE_Q=$Q DEFMM_TILE_K=$K DEFMM_TILE_OPS=$OPS DEFMM_TILE_EV=$EV timeout 300 $B --m2l-levels tiles > gpurun_out/st_${Q}_${K}_${OPS}_${EV}.log 2>&1
done; done; done; done
python - > gpurun_out/st_summary.txt <<'PY'
import json, glob
for f in sorted(glob.glob("gpurun_out/st_*.log")):
    l=[x for x in open(f) if x.startswith("{")]
    if not l: print(f, "no line"); continue
    d=json.loads(l[-1])
    print(f, round(d["ms_per_step"],3), d.get("isolated_ms"), d["accuracy"]["rel_l2_vs_direct_1000"])
PY
