# round-1 GPU pass 21: config 5 bench at full size
set -x
timeout 900 python bench.py --config c5 --steps 5 --warmup 3 > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err
cat gpurun_out/bench_c5.json; tail -5 gpurun_out/bench_c5.err; nvidia-smi --query-gpu=memory.used,memory.total --format=csv
