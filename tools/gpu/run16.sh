# round-1 GPU pass 16: window gather variants (window size, register budget)
set -x
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider -x 2>&1 | tail -40 > gpurun_out/pytest_gpu.txt
for v in "280 3" "280 4" "540 2" "540 3" "160 4"; do set -- $v
  FF_WIN_ELEMS=$1 FF_WMINB=$2 timeout 400 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/bench_win_$1_$2.json 2>/dev/null
done
FF_WIN_ELEMS=280 FF_WMINB=3 timeout 600 ncu --set full --clock-control none --import-source on -k regex:ff_gather_windows -s 1 -c 1 -o gpurun_out/prof_win2 \
  python bench.py --steps 2 --warmup 1 --e2e-steps 0 --no-cpu-baseline > gpurun_out/ncu_full.txt 2>&1
grep -E "passed|failed|Error|assert" gpurun_out/pytest_gpu.txt | head
for f in gpurun_out/bench_win_*.json; do echo $f $(python -c "import json;d=json.load(open('$f'));g=d['config']['gather_plan'];print(d['ms_per_step'],g['window_rows'],g['window_max_elems'])"); done
