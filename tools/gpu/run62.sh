# round-1 final artifacts (2-warp class CTAs)
nvidia-smi --query-gpu=name,clocks.max.sm,memory.total --format=csv,noheader; nproc
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider 2>&1 | tail -3 > gpurun_out/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1
timeout 600 python bench.py --steps 20 --warmup 3 > gpurun_out/bench_ns.json 2> gpurun_out/bench_ns.err
timeout 600 python bench.py --steps 20 --warmup 3 --scatter atomic --no-cpu-baseline > gpurun_out/bench_ns_atomic.json 2> gpurun_out/bench_ns_atomic.err
for c in c3 c2 c1 c4; do timeout 400 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; done
timeout 900 python bench.py --config c5 --steps 5 --warmup 3 > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
cat gpurun_out/pytest_gpu.txt; tail -1 gpurun_out/smoke.txt | cut -c1-120
for f in ns ns_atomic c3 c2 c1 c4 c5 ref; do echo "$f: $(python -c "import json;d=json.load(open('gpurun_out/bench_$f.json'));print(round(d['ms_per_step'],4),d['value'],d.get('roofline',{}).get('frac'),d.get('gpu_launches'),d.get('clocks',{}).get('reasons'))" 2>&1 | tail -1)"; done
