# round-1 GPU pass 26: fused class kernel default; full tests; profile
set -x
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider 2>&1 | tail -30 > gpurun_out/pytest_gpu.txt
timeout 400 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/bench_ns.json 2> gpurun_out/bench_ns.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:ff_gather_classes -s 1 -c 1 -o gpurun_out/prof_fused \
  python bench.py --steps 2 --warmup 1 --e2e-steps 0 --no-cpu-baseline > gpurun_out/ncu_full.txt 2>&1
grep -E "passed|failed|Error|assert" gpurun_out/pytest_gpu.txt | head
python -c "import json;d=json.load(open('gpurun_out/bench_ns.json'));print(d['ms_per_step'],d['config']['k2a_ms'],d['config']['k2_ms'],d['roofline']['frac'])"
