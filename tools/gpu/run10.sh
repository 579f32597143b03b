# round-1 GPU pass 10: class kernels with next-item prefetch, big classes only
set -x
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider -x 2>&1 | tail -30 > gpurun_out/pytest_gpu.txt
timeout 400 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/bench_ns.json 2> gpurun_out/bench_ns.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:ff_gather -s 4 -c 4 -o gpurun_out/prof_gather_ns9 \
  python bench.py --steps 2 --warmup 1 --e2e-steps 0 --no-cpu-baseline > gpurun_out/ncu_full.txt 2>&1
grep -E "passed|failed|Error|assert" gpurun_out/pytest_gpu.txt | head; cat gpurun_out/bench_ns.json; tail -3 gpurun_out/bench_ns.err; tail -2 gpurun_out/ncu_full.txt
