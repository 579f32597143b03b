# vector gather: CTA per component pair, write-back stores
timeout 1500 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "elasticity" -p no:cacheprovider --durations=3 2>&1 | tail -8
for v in FF_NONE=1 FF_IPW=1 FF_VDEPTH=1 FF_VDEPTH=4; do
  echo "$v $(env $v timeout 600 python bench.py --config c5 --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 0 | python -c "import json,sys;d=json.load(sys.stdin);print(round(d['ms_per_step'],3), d['config'].get('k2_ms'), d['config'].get('k2a_ms'), d['roofline']['frac'])")"
done
