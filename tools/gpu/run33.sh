# round-1 GPU pass 33: final round artifacts (class gather: fused, L1 no-allocate, prefetch)
set -x
nvidia-smi --query-gpu=name,clocks.max.sm,memory.total --format=csv; nproc
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider 2>&1 | tail -4 > gpurun_out/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1
timeout 600 python bench.py --steps 20 --warmup 3 > gpurun_out/bench_ns.json 2> gpurun_out/bench_ns.err
for c in c3 c2 c1 c4; do timeout 400 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; done
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_ns_gather.csv \
  python bench.py --steps 2 --warmup 1 --e2e-steps 0 --no-cpu-baseline > gpurun_out/ncu_launch_bench.txt 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:ff_gather_classes -s 1 -c 1 -o gpurun_out/prof_cls_final3 \
  python bench.py --steps 2 --warmup 1 --e2e-steps 0 --no-cpu-baseline > gpurun_out/ncu_full.txt 2>&1
tail -2 gpurun_out/pytest_gpu.txt; tail -1 gpurun_out/smoke.txt | cut -c1-150
for f in ns c3 c2 c1 c4; do echo "$f: $(python -c "import json;d=json.load(open('gpurun_out/bench_$f.json'));print(d['ms_per_step'],d['value'],d['roofline']['frac'],d['config']['scatter'])")"; done
