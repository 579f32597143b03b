# ablation on the final round-1 class kernel (timing only)
for v in FF_NONE=1 FF_ABLATE_NOWRITE=1 FF_ABLATE_NOG=1 FF_ABLATE_NOB=1 "FF_ABLATE_NOG=1 FF_ABLATE_NOB=1" "FF_ABLATE_NOWRITE=1 FF_ABLATE_NOG=1 FF_ABLATE_NOB=1"; do
  echo "$v $(env $v timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 0 2>/dev/null | python -c "import json,sys;d=json.load(sys.stdin);print(round(d['ms_per_step'],4), round(d['config']['k2_ms'],4))")"
done
