# round-1 GPU pass 30: next-item header/record prefetch in the class gather
set -x
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -x -k "gather or class or north or elasticity" 2>&1 | tail -3 > gpurun_out/pytest_gpu.txt
for v in "2 3" "4 3" "1 3"; do set -- $v
  FF_IPW=$1 FF_MINB_S=$2 timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/b30.json 2>/dev/null
  echo "ipw=$1 minb=$2 $(python -c "import json;d=json.load(open('gpurun_out/b30.json'));print(d['ms_per_step'],d['config']['k2_ms'])")"
done
grep -E "passed|failed" gpurun_out/pytest_gpu.txt
