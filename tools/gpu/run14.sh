# round-1 GPU pass 14: Morton element order for per-element records; write-out row loop
set -x
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider -x 2>&1 | tail -40 > gpurun_out/pytest_gpu.txt
timeout 400 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/bench_ns_eo.json 2>/dev/null
FF_NO_EORDER=1 timeout 400 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/bench_ns_noeo.json 2>/dev/null
FF_IPW=1 timeout 400 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/bench_ns_eo_ipw1.json 2>/dev/null
timeout 600 ncu --set full --clock-control none --import-source on -k regex:ff_gather -s 4 -c 4 -o gpurun_out/prof_eo \
  python bench.py --steps 2 --warmup 1 --e2e-steps 0 --no-cpu-baseline > gpurun_out/ncu_full.txt 2>&1
grep -E "passed|failed|Error|assert" gpurun_out/pytest_gpu.txt | head
for f in gpurun_out/bench_ns_eo.json gpurun_out/bench_ns_noeo.json gpurun_out/bench_ns_eo_ipw1.json; do echo $f $(python -c "import json;d=json.load(open('$f'));print(d['ms_per_step'],d['config']['k2a_ms'],d['config']['k2_ms'])"); done
