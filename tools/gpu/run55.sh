FF_CD_GROUP=1 timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "elasticity_class" -p no:cacheprovider 2>&1 | tail -1
for v in FF_NONE=1 FF_CD_GROUP=1 "FF_CD_GROUP=1 FF_IPW=2"; do
  echo "c5 $v $(env $v timeout 600 python bench.py --config c5 --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 0 | python -c "import json,sys;d=json.load(sys.stdin);print(round(d['ms_per_step'],3), d['config'].get('k2_ms'))")"
done
