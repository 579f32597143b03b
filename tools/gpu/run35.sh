# upper bound of K2a/class overlap (FF_K2A_RACE: timing only), generic-side default
for i in 1 2; do
for v in FF_GENERIC_SERIAL=1 FF_NONE=1 FF_K2A_RACE=1; do
  echo "$v $(env $v timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 0 | python -c "import json,sys;d=json.load(sys.stdin);print(round(d['ms_per_step'],4))")"
done; done
