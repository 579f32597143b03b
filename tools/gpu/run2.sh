# round-1 GPU pass 2: tests, bench lines, ncu launch list + full capture of K2
set -x
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider 2>&1 | tail -15 > gpurun_out/pytest_gpu.txt
for c in ns c3 c2 c1; do
  timeout 600 python bench.py --config $c --steps 20 --warmup 3 $([ $c != ns ] && echo --no-cpu-baseline) > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_ns.csv \
  python bench.py --steps 2 --warmup 1 --e2e-steps 0 --no-cpu-baseline > gpurun_out/ncu_launch_bench.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:ff_assemble -s 2 -c 1 -o gpurun_out/prof_k2_ns \
  python bench.py --steps 2 --warmup 1 --e2e-steps 0 --no-cpu-baseline > gpurun_out/ncu_full.txt 2>&1
tail -3 gpurun_out/pytest_gpu.txt; for c in ns c3 c2 c1; do cat gpurun_out/bench_$c.json; tail -2 gpurun_out/bench_$c.err; done; tail -5 gpurun_out/ncu_full.txt
