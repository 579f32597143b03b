# GPU pass 3: row-tile scatter parity + bench + ncu
set -x
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -x 2>&1 | tail -15 > gpurun_out/pytest_gpu.txt
timeout 600 python bench.py --steps 20 --warmup 3 > gpurun_out/bench_ns.json 2> gpurun_out/bench_ns.err
for c in c3 c2 c1; do timeout 600 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:ff_assemble_rowtile -s 2 -c 1 -o gpurun_out/prof_rt_ns \
  python bench.py --steps 2 --warmup 1 --e2e-steps 0 --no-cpu-baseline > gpurun_out/ncu_full.txt 2>&1
tail -3 gpurun_out/pytest_gpu.txt; for c in ns c3 c2 c1; do cat gpurun_out/bench_$c.json; tail -3 gpurun_out/bench_$c.err; done; tail -3 gpurun_out/ncu_full.txt
