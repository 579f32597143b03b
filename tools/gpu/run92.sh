timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "gather or class or isolated or graph or elasticity" -p no:cacheprovider 2>&1 | tail -1 > gpurun_out/t92.txt
for c in ns c3 c2 c5; do
  st=20; [ $c = c5 ] && st=5
  echo "$c $(timeout 600 python bench.py --config $c --steps $st --warmup 3 --no-cpu-baseline --e2e-steps 0 2>/dev/null | python -c "import json,sys;d=json.load(sys.stdin);print(round(d['ms_per_step'],4))")"
done
cat gpurun_out/t92.txt
