# round-1 GPU pass 11: class kernel variants (items per warp, register budgets)
set -x
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider -x 2>&1 | tail -40 > gpurun_out/pytest_gpu.txt
for v in "4 4 2" "1 4 2" "2 4 2" "1 5 2" "1 4 1" "8 4 2"; do set -- $v
  FF_IPW=$1 FF_MINB_S=$2 FF_MINB_L=$3 timeout 400 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/bench_ns_$1_$2_$3.json 2>/dev/null
  echo "ipw=$1 minb_s=$2 minb_l=$3 $(python -c "import json;d=json.load(open('gpurun_out/bench_ns_$1_$2_$3.json'));print(d['ms_per_step'],d['config']['k2a_ms'],d['config']['k2_ms'])")"
done
grep -E "passed|failed|Error|assert" gpurun_out/pytest_gpu.txt | head
