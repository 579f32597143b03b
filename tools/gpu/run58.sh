# cross-item record prefetch before the write-out
FF_XPRE=1 timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "class or gather or isolated" -p no:cacheprovider 2>&1 | tail -1
for i in 1 2; do for v in FF_NONE=1 FF_XPRE=1 "FF_XPRE=1 FF_MINB_S=2" "FF_XPRE=1 FF_IPW=4"; do
  echo "$v $(env $v timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 0 | python -c "import json,sys;d=json.load(sys.stdin);print(round(d['ms_per_step'],4), d['config'].get('k2_ms'))")"
done; done
