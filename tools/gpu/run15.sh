# round-1 GPU pass 15: window row gather (element records in shared memory)
set -x
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider -x 2>&1 | tail -40 > gpurun_out/pytest_gpu.txt
timeout 400 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/bench_ns_win.json 2>gpurun_out/bench_ns_win.err
FF_NO_WINDOWS=1 timeout 400 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/bench_ns_nowin.json 2>/dev/null
timeout 600 ncu --set full --clock-control none --import-source on -k regex:ff_gather_windows -s 1 -c 1 -o gpurun_out/prof_win \
  python bench.py --steps 2 --warmup 1 --e2e-steps 0 --no-cpu-baseline > gpurun_out/ncu_full.txt 2>&1
grep -E "passed|failed|Error|assert" gpurun_out/pytest_gpu.txt | head
for f in gpurun_out/bench_ns_win.json gpurun_out/bench_ns_nowin.json; do echo $f $(python -c "import json;d=json.load(open('$f'));print(d['ms_per_step'],d['config']['k2a_ms'],d['config']['k2_ms'],d['config']['gather_plan'])"); done
tail -3 gpurun_out/bench_ns_win.err
