# round-1 GPU pass 17: concurrent short/long class kernels; window gather opt-in
set -x
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider -x 2>&1 | tail -40 > gpurun_out/pytest_gpu.txt
timeout 400 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/bench_ns_conc.json 2>gpurun_out/bench_ns_conc.err
FF_SERIAL_CLASSES=1 timeout 400 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/bench_ns_serial.json 2>/dev/null
grep -E "passed|failed|Error|assert" gpurun_out/pytest_gpu.txt | head
for f in gpurun_out/bench_ns_conc.json gpurun_out/bench_ns_serial.json; do echo $f $(python -c "import json;d=json.load(open('$f'));print(d['ms_per_step'],d['config']['k2a_ms'],d['config']['k2_ms'])"); done
tail -3 gpurun_out/bench_ns_conc.err
