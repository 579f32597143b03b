# padded [nv][4] coordinates: one 256-bit load per vertex in the element kernels
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider 2>&1 | tail -1 > gpurun_out/t71.txt
for c in ns c2 c3 c4 c5; do
  st=20; [ $c = c5 ] && st=5
  echo "$c $(timeout 600 python bench.py --config $c --steps $st --warmup 3 --no-cpu-baseline --e2e-steps 0 2>/dev/null | python -c "import json,sys;d=json.load(sys.stdin);print(round(d['ms_per_step'],4), d['config'].get('k2a_ms'), d['config'].get('k2_ms'))")"
done
timeout 300 python bench.py --steps 20 --warmup 3 --scatter atomic --no-cpu-baseline --e2e-steps 0 2>/dev/null | python -c "import json,sys;d=json.load(sys.stdin);print('ns atomic', round(d['ms_per_step'],4), d['config'].get('k2_ms'))"
cat gpurun_out/t71.txt
