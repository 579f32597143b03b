# round-1 GPU pass 27: L1 no-allocate element-record loads
set -x
for v in "0" "1"; do
  if [ $v = 1 ]; then export FF_EINV_NA=1; else unset FF_EINV_NA; fi
  timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/b27_$v.json 2>/dev/null
  echo "na=$v $(python -c "import json;d=json.load(open('gpurun_out/b27_$v.json'));print(d['ms_per_step'],d['config']['k2_ms'])")"
  FF_IPW=2 timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/b27_$v.json 2>/dev/null
  echo "na=$v ipw2 $(python -c "import json;d=json.load(open('gpurun_out/b27_$v.json'));print(d['ms_per_step'],d['config']['k2_ms'])")"
done
