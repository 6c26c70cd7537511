# A/B timing of library variants (tools/variant_build.py): bench config 2 and the config-4 frame per variant
set +e
V=paper_2311_11700_b200/build/variants
for v in "$@"; do
  for c in 2 4; do
    if [ $c = 4 ]; then X="--config 4 --frame"; else X=""; fi
    if [ $v = base ]; then L=""; else L=$V/libgs_$v.so; fi
    GS_LIB=$L timeout 300 python bench.py $X --no-cpu-baseline --no-e2e --steps 30 --warmup 10 2>/dev/null | tail -1 | python -c "
import json,sys;d=json.loads(sys.stdin.read());k=d['kernels_ms_per_step'];print('$v','c$c',round(d['ms_per_step'],4),' '.join(f'{a[:10]}={b*1000:.1f}' for a,b in k.items()))"
  done
done
