# round-1 GPU pass 25: fused class kernel (long rows in slot passes)
set -x
FF_FUSED_CLASSES=1 timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -x -k "gather or class or north" 2>&1 | tail -5 > gpurun_out/pytest_gpu.txt
for v in "0 4" "1 4" "1 3"; do set -- $v
  if [ $1 = 1 ]; then export FF_FUSED_CLASSES=1; else unset FF_FUSED_CLASSES; fi
  FF_MINB_S=$2 timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/b25_$1_$2.json 2>/dev/null
  echo "fused=$1 minb_s=$2 $(python -c "import json;d=json.load(open('gpurun_out/b25_$1_$2.json'));print(d['ms_per_step'],d['config']['k2_ms'])")"
done
grep -E "passed|failed" gpurun_out/pytest_gpu.txt
