set -x
nvidia-smi --query-gpu=name,clocks.max.sm,memory.total --format=csv; nproc; lscpu | grep "Model name"; free -g | head -2
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider 2>&1 | tail -40 > gpurun_out/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1
timeout 600 python bench.py --steps 20 --warmup 3 > gpurun_out/bench_ns.json 2> gpurun_out/bench_ns.err
tail -3 gpurun_out/pytest_gpu.txt; cat gpurun_out/smoke.txt | tail -3; cat gpurun_out/bench_ns.json; tail -5 gpurun_out/bench_ns.err
