for i in 1 2; do for v in FF_NONE=1 FF_CLASS_PRIO=1; do
  echo "ns $v $(env $v timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 0 2>/dev/null | python -c "import json,sys;d=json.load(sys.stdin);print(round(d['ms_per_step'],4))")"
done; done
for v in FF_NONE=1 FF_CLASS_PRIO=1; do
  echo "c3 $v $(env $v timeout 300 python bench.py --config c3 --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 0 2>/dev/null | python -c "import json,sys;d=json.load(sys.stdin);print(round(d['ms_per_step'],4))")"
done
