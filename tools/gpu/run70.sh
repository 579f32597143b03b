# CUDA-graph replay of the assembly launch sequence
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider 2>&1 | tail -1 > gpurun_out/t70.txt
for c in c1 c2 c3 ns c5; do for v in FF_NONE=1 FF_NO_GRAPH=1; do
  st=20; [ $c = c5 ] && st=5
  echo "$c $v $(env $v timeout 600 python bench.py --config $c --steps $st --warmup 3 --no-cpu-baseline --e2e-steps 0 2>/dev/null | python -c "import json,sys;d=json.load(sys.stdin);print(round(d['ms_per_step'],4), d['config'].get('k2a_ms'), d['config'].get('k2_ms'))")"
done; done
cat gpurun_out/t70.txt
