# vector (elasticity) row gather: parity + C5 bench + class kernel profile
timeout 1500 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "elasticity" -p no:cacheprovider --durations=5 2>&1 | tail -30 > gpurun_out/t42.txt
tail -12 gpurun_out/t42.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:ff_gather_classes -s 1 -c 1 -o gpurun_out/prof_c5cls \
  python bench.py --config c5 --steps 1 --warmup 1 --e2e-steps 0 --no-cpu-baseline > gpurun_out/ncu_c5.txt 2>&1
tail -2 gpurun_out/ncu_c5.txt
