# asynchronous record staging (cp.async) in the class kernel
for a in 2 4; do FF_CLASS_ASYNC=$a timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "class or gather" -p no:cacheprovider 2>&1 | tail -1; done
for v in FF_NONE=1 FF_CLASS_ASYNC=2 FF_CLASS_ASYNC=3 FF_CLASS_ASYNC=4 "FF_CLASS_ASYNC=2 FF_MINB_S=4" "FF_CLASS_ASYNC=4 FF_MINB_S=2" "FF_CLASS_ASYNC=2 FF_IPW=4" "FF_CLASS_ASYNC=4 FF_IPW=4"; do
  echo "$v $(env $v timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 0 | python -c "import json,sys;d=json.load(sys.stdin);print(round(d['ms_per_step'],4), d['config'].get('k2_ms'))")"
done
