set +e
V=paper_2311_11700_b200/build/variants
for v in "$@"; do
  for c in 2 4; do
    if [ $c = 4 ]; then X="--config 4 --frame"; else X=""; fi
    GS_LIB=$V/libgs_$v.so timeout 300 python bench.py $X --no-cpu-baseline --no-e2e --steps 30 --warmup 10 2>/dev/null | tail -1 | python -c "
import json,sys;d=json.loads(sys.stdin.read());k=d['kernels_ms_per_step'];print('$v','c$c',round(d['ms_per_step'],4),k.get('bucket_emit'),k.get('bin_coop'))"
  done
done
