# round-1 GPU pass 24: class kernel register budget / items-per-warp sweep
set -x
for v in "4 4" "4 5" "4 6" "1 5" "2 6" "8 5"; do set -- $v
  FF_IPW=$1 FF_MINB_S=$2 timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/b24_$1_$2.json 2>/dev/null
  echo "ipw=$1 minb_s=$2 $(python -c "import json;d=json.load(open('gpurun_out/b24_$1_$2.json'));print(d['ms_per_step'],d['config']['k2_ms'])")"
done
