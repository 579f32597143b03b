# round-1 GPU pass 5: row-gather scatter parity + bench + launch list + ncu
set -x
nvidia-smi --query-gpu=name,clocks.max.sm,memory.total --format=csv; nproc
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider -x 2>&1 | tail -25 > gpurun_out/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1
timeout 400 python bench.py --steps 20 --warmup 3 > gpurun_out/bench_ns.json 2> gpurun_out/bench_ns.err
for c in c3 c2 c1; do timeout 300 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_ns_gather.csv \
  python bench.py --steps 2 --warmup 1 --e2e-steps 0 --no-cpu-baseline > gpurun_out/ncu_launch_bench.txt 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:ff_gather -s 2 -c 2 -o gpurun_out/prof_gather_ns \
  python bench.py --steps 2 --warmup 1 --e2e-steps 0 --no-cpu-baseline > gpurun_out/ncu_full.txt 2>&1
tail -25 gpurun_out/pytest_gpu.txt; tail -2 gpurun_out/smoke.txt; for c in ns c3 c2 c1; do cat gpurun_out/bench_$c.json; tail -3 gpurun_out/bench_$c.err; done; tail -3 gpurun_out/ncu_full.txt
