W=$1; shift
for L in none "$@"; do
  if [ "$L" = none ]; then E=""; else E="$L"; fi
  DEFMM_M2L_LEVELS="$E" timeout 400 python bench.py --workload $W --steps 5 --warmup 2 --no-cpu-baseline --no-graph > gpurun_out/lv.log 2>&1
  python -c "
import json
l=[x for x in open('gpurun_out/lv.log') if x.startswith('{')]
d=json.loads(l[-1]) if l else {}
print('$W', '$L', round(d.get('stages_ms',{}).get('m2l',-1),3), (d.get('c128_same_lists') or d.get('c64_same_lists') or {}).get('m2l_ms'))
" >> gpurun_out/lvexp.txt
done
