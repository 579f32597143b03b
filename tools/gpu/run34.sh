# generic rows on the side stream, concurrent with the class kernel
for i in 1 2; do
for v in "" 1; do
  echo "FF_GENERIC_SIDE=$v $(env ${v:+FF_GENERIC_SIDE=$v} timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 0 | python -c "import json,sys;d=json.load(sys.stdin);print(round(d['ms_per_step'],4))")"
done; done
