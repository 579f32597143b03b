# round-1 GPU pass 9: single class kernel with slot-range passes
set -x
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider -x 2>&1 | tail -30 > gpurun_out/pytest_gpu.txt
timeout 400 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/bench_ns.json 2> gpurun_out/bench_ns.err
FF_CLASS_MINB=3 timeout 400 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/bench_ns_mb3.json 2> gpurun_out/bench_ns_mb3.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:ff_gather_classes -s 1 -c 1 -o gpurun_out/prof_gather_ns8 \
  python bench.py --steps 2 --warmup 1 --e2e-steps 0 --no-cpu-baseline > gpurun_out/ncu_full.txt 2>&1
grep -E "passed|failed" gpurun_out/pytest_gpu.txt; cat gpurun_out/bench_ns.json; cat gpurun_out/bench_ns_mb3.json; tail -3 gpurun_out/bench_ns.err; tail -2 gpurun_out/ncu_full.txt
