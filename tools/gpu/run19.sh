# round-1 GPU pass 19: pointwise element body as a runtime quadrature loop (C4)
set -x
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider -x 2>&1 | tail -30 > gpurun_out/pytest_gpu.txt
timeout 400 python bench.py --config c4 --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err
grep -E "passed|failed|Error|assert" gpurun_out/pytest_gpu.txt | head
cut -c1-300 gpurun_out/bench_c4.json; python -c "import json;d=json.load(open('gpurun_out/bench_c4.json'));print(d['ms_per_step'],d['config']['k0_ms'],d['config']['k2_ms'],d['config']['registers'],d['config']['flops_per_element'])"
tail -3 gpurun_out/bench_c4.err
