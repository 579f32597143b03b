timeout 2000 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=5 2>&1 | tail -9 > gpurun_out/pytest_gpu.txt
cat gpurun_out/pytest_gpu.txt
timeout 900 python bench.py --config c5 --steps 5 --warmup 3 > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err
timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/bench_ns_q.json
for f in c5 ns_q; do echo "$f $(python -c "import json;d=json.load(open('gpurun_out/bench_$f.json'));print(d['ms_per_step'],d['roofline']['frac'],d['config']['scatter'])")"; done
