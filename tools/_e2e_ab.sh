set +e
V=paper_2311_11700_b200/build/variants
for v in "$@"; do
  if [ $v = base ]; then L=""; else L=$V/libgs_$v.so; fi
  GS_LIB=$L timeout 300 python bench.py --no-cpu-baseline --steps 50 --warmup 10 2>/dev/null | tail -1 | python -c "
import json,sys;d=json.loads(sys.stdin.read());print('$v',round(d['ms_per_step'],4),'e2e',round(d['e2e']['value'],1))"
done
