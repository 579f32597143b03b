set -x
for v in 0.005 0.0009 0.0003; do
  FF_CLASS_FRAC=$v timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/b32.json 2>/dev/null
  echo "frac=$v $(python -c "import json;d=json.load(open('gpurun_out/b32.json'));g=d['config']['gather_plan'];print(d['ms_per_step'],d['config']['k2_ms'],g['n_classes'],g['n_class_rows'])")"
done
