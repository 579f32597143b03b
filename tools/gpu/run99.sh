timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider 2>&1 | tail -1 > gpurun_out/t99.txt
for c in ns c3 c2 c1 c5; do
  st=20; [ $c = c5 ] && st=5
  echo "$c $(timeout 600 python bench.py --config $c --steps $st --warmup 3 --no-cpu-baseline --e2e-steps 0 2>/dev/null | python -c "import json,sys;d=json.load(sys.stdin);print(round(d['ms_per_step'],4))")"
done
cat gpurun_out/t99.txt
