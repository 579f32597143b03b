for v in "FF_IPW=1 FF_MINB_S=3" "FF_IPW=1 FF_VDEPTH=1" "FF_IPW=1 FF_VDEPTH=1 FF_MINB_S=3" "FF_IPW=1 FF_EINV_L1=1"; do
  echo "$v $(env $v timeout 600 python bench.py --config c5 --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 0 | python -c "import json,sys;d=json.load(sys.stdin);print(round(d['ms_per_step'],3), d['config'].get('k2_ms'), d['config'].get('k2a_ms'), d['roofline']['frac'])")"
done
