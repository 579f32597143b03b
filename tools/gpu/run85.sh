for c in ns c3; do for v in FF_ITEM_WINDOW=16384 FF_ITEM_WINDOW=65536 FF_ITEM_WINDOW=262144 FF_ITEM_WINDOW=1048576; do
  echo "$c $v $(env $v timeout 300 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 0 2>/dev/null | python -c "import json,sys;d=json.load(sys.stdin);print(round(d['ms_per_step'],4))")"
done; done
