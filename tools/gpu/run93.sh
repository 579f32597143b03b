timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "class or isolated" -p no:cacheprovider 2>&1 | tail -1 > gpurun_out/t93.txt
for i in 1 2; do for c in ns c3; do
  echo "$c $(timeout 300 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 0 2>/dev/null | python -c "import json,sys;d=json.load(sys.stdin);print(round(d['ms_per_step'],4))")"
done; done
cat gpurun_out/t93.txt
