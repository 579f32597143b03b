timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c1.csv \
  python bench.py --config c1 --steps 2 --warmup 1 --e2e-steps 0 --no-cpu-baseline > /dev/null 2>&1
python - <<'PY'
import csv
rows=[r for r in csv.DictReader(l for l in open('gpurun_out/launches_c1.csv') if not l.startswith('=='))]
ff=[(r['Kernel Name'][:30], float(r['Metric Value'])) for r in rows if r['Kernel Name'].startswith('ff_')]
for k,v in ff[-8:]: print(k, v)
PY
