for v in FF_NONE=1 FF_IPW=3 "FF_CWARPS=3 FF_MINB_S=4" FF_ITEM_WINDOW=8192 FF_ITEM_WINDOW=32768 "FF_CWARPS=1 FF_MINB_S=12 FF_IPW=4"; do
  echo "ns $v $(env $v timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 0 2>/dev/null | python -c "import json,sys;d=json.load(sys.stdin);print(round(d['ms_per_step'],4))")"
done
