for c in c2 c1 c3; do for v in FF_NONE=1 FF_WINDOWS=1; do
  echo "$c $v $(env $v timeout 300 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 0 2>/dev/null | python -c "import json,sys;d=json.load(sys.stdin);print(round(d['ms_per_step'],4), d['config'].get('k2a_ms'), d['config'].get('k2_ms'))")"
done; done
timeout 300 python bench.py --config c2 --scatter atomic --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 0 2>/dev/null | python -c "import json,sys;d=json.load(sys.stdin);print('c2 atomic', round(d['ms_per_step'],4), d['config'].get('k0_ms'), d['config'].get('k2_ms'))"
