# round-1 GPU pass 18: round artifacts for the class-specialised row gather
set -x
nvidia-smi --query-gpu=name,clocks.max.sm,memory.total --format=csv; nproc
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider 2>&1 | tail -6 > gpurun_out/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1
timeout 600 python bench.py --steps 20 --warmup 3 > gpurun_out/bench_ns.json 2> gpurun_out/bench_ns.err
timeout 400 python bench.py --steps 20 --warmup 3 --scatter atomic --no-cpu-baseline --e2e-steps 0 > gpurun_out/bench_ns_atomic.json 2> /dev/null
for c in c3 c2 c1 c4; do timeout 400 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; done
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_ns_gather.csv \
  python bench.py --steps 2 --warmup 1 --e2e-steps 0 --no-cpu-baseline > gpurun_out/ncu_launch_bench.txt 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:ff_gather_classes_s -s 1 -c 1 -o gpurun_out/prof_cls_s_final \
  python bench.py --steps 2 --warmup 1 --e2e-steps 0 --no-cpu-baseline > gpurun_out/ncu_full.txt 2>&1
tail -3 gpurun_out/pytest_gpu.txt; tail -1 gpurun_out/smoke.txt | cut -c1-200
for f in ns ns_atomic c3 c2 c1 c4 ref; do echo "$f: $(cut -c1-400 gpurun_out/bench_$f.json)"; done
