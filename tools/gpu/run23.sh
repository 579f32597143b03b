# round-1 GPU pass 23: 256-bit record loads, SoA load vectors, private NVRTC 12.9
set -x
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -x 2>&1 | tail -30 > gpurun_out/pytest_gpu.txt
timeout 400 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/bench_ns.json 2> gpurun_out/bench_ns.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:ff_gather -s 5 -c 5 -o gpurun_out/prof_r23 \
  python bench.py --steps 2 --warmup 1 --e2e-steps 0 --no-cpu-baseline > gpurun_out/ncu_full.txt 2>&1
grep -E "passed|failed|Error|assert" gpurun_out/pytest_gpu.txt | head
python -c "import json;d=json.load(open('gpurun_out/bench_ns.json'));print(d['ms_per_step'],d['config']['k2a_ms'],d['config']['k2_ms'],d['roofline']['frac'])"
tail -3 gpurun_out/bench_ns.err
