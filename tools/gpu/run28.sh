# round-1 GPU pass 28: items per warp / register budget with no-allocate loads
set -x
for v in "1 3" "2 3" "3 3" "4 3" "2 2" "2 4"; do set -- $v
  FF_IPW=$1 FF_MINB_S=$2 timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/b28.json 2>/dev/null
  echo "ipw=$1 minb=$2 $(python -c "import json;d=json.load(open('gpurun_out/b28.json'));print(d['ms_per_step'],d['config']['k2_ms'])")"
done
