timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider 2>&1 | tail -1 > gpurun_out/t88.txt
for i in 1 2; do for c in ns c3 c2; do
  echo "$c $(timeout 300 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 0 2>/dev/null | python -c "import json,sys;d=json.load(sys.stdin);print(round(d['ms_per_step'],4), round(d['config']['k2a_ms'],4))")"
done; done
cat gpurun_out/t88.txt
