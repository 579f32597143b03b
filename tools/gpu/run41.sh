# vector (elasticity) row gather: parity + C5 bench
timeout 1200 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "elasticity" -p no:cacheprovider 2>&1 | tail -30 > gpurun_out/t41.txt
timeout 900 python bench.py --config c5 --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/b41_c5.json 2> gpurun_out/b41_c5.err
tail -5 gpurun_out/t41.txt; tail -3 gpurun_out/b41_c5.err
python -c "import json;d=json.load(open('gpurun_out/b41_c5.json'));print(d['ms_per_step'],d['config']['scatter'],d['config'].get('k2_ms'),d['config'].get('k2a_ms'),d['config'].get('nvrtc_compile_ms'),d['roofline']['frac'])"
