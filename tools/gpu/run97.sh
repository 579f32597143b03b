for v in FF_NONE=1 FF_MINB_S=2 FF_IPW=2 FF_VDEPTH=1 FF_VDEPTH=3; do
  echo "c5 $v $(env $v timeout 600 python bench.py --config c5 --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 0 2>/dev/null | python -c "import json,sys;d=json.load(sys.stdin);print(round(d['ms_per_step'],3))")"
done
