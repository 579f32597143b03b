# round-1 GPU pass 6: Morton-window gather plan, coalesced K2a, 2-step MLP
set -x
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider -x 2>&1 | tail -15 > gpurun_out/pytest_gpu.txt
timeout 400 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/bench_ns.json 2> gpurun_out/bench_ns.err
timeout 300 python bench.py --config c2 --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:ff_gather -s 2 -c 2 -o gpurun_out/prof_gather_ns2 \
  python bench.py --steps 2 --warmup 1 --e2e-steps 0 --no-cpu-baseline > gpurun_out/ncu_full.txt 2>&1
tail -15 gpurun_out/pytest_gpu.txt; for c in ns c2; do cat gpurun_out/bench_$c.json; tail -3 gpurun_out/bench_$c.err; done; tail -3 gpurun_out/ncu_full.txt
