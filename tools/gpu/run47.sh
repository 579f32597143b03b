timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "class or elasticity" -p no:cacheprovider 2>&1 | tail -1
for c in ns c5; do
  echo "$c $(timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 0 | python -c "import json,sys;d=json.load(sys.stdin);print(round(d['ms_per_step'],3), d['config'].get('k2_ms'), d['roofline']['frac'])")"
done
