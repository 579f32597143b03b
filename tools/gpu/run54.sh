# round-1 final artifacts (single-pass class gather, vector sub-row gather, weak scaling)
nvidia-smi --query-gpu=name,clocks.max.sm,memory.total --format=csv; nproc
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider 2>&1 | tail -3 > gpurun_out/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1
timeout 600 python bench.py --steps 20 --warmup 3 > gpurun_out/bench_ns.json 2> gpurun_out/bench_ns.err
timeout 600 python bench.py --steps 20 --warmup 3 --scatter atomic --no-cpu-baseline > gpurun_out/bench_ns_atomic.json 2> gpurun_out/bench_ns_atomic.err
for c in c3 c2 c1 c4; do timeout 400 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; done
timeout 900 python bench.py --config c5 --steps 5 --warmup 3 > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_ns_gather.csv \
  python bench.py --steps 2 --warmup 1 --e2e-steps 0 --no-cpu-baseline > gpurun_out/ncu_launch_bench.txt 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:ff_gather_classes -s 1 -c 1 -o gpurun_out/prof_final_r1 \
  python bench.py --steps 2 --warmup 1 --e2e-steps 0 --no-cpu-baseline > gpurun_out/ncu_full.txt 2>&1
cat gpurun_out/pytest_gpu.txt; tail -1 gpurun_out/smoke.txt | cut -c1-150
for f in ns ns_atomic c3 c2 c1 c4 c5 ref; do echo "$f: $(python -c "import json;d=json.load(open('gpurun_out/bench_$f.json'));print(d['ms_per_step'],d['value'],d.get('roofline',{}).get('frac'),d.get('config',{}).get('scatter'))" 2>&1 | tail -1)"; done
