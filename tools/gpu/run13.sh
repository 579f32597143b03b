# round-1 GPU pass 13: class-grouped CTAs, shared write-out (instruction footprint)
set -x
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider -x 2>&1 | tail -40 > gpurun_out/pytest_gpu.txt
for v in "4 4 2" "1 4 2" "8 4 2"; do set -- $v
  FF_IPW=$1 FF_MINB_S=$2 FF_MINB_L=$3 timeout 400 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/bench_ns_$1_$2_$3.json 2>/dev/null
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:ff_gather_classes -s 2 -c 2 -o gpurun_out/prof_cls2 \
  python bench.py --steps 2 --warmup 1 --e2e-steps 0 --no-cpu-baseline > gpurun_out/ncu_full.txt 2>&1
grep -E "passed|failed|Error|assert" gpurun_out/pytest_gpu.txt | head
for f in gpurun_out/bench_ns_*_*_*.json; do echo $f $(python -c "import json;d=json.load(open('$f'));print(d['ms_per_step'],d['config']['k2a_ms'],d['config']['k2_ms'])"); done
