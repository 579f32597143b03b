FF_CLASS_ASYNC=2 timeout 600 ncu --set full --clock-control none --import-source on -k regex:ff_gather_classes -s 1 -c 1 -o gpurun_out/prof_async2 \
  python bench.py --steps 2 --warmup 1 --e2e-steps 0 --no-cpu-baseline > gpurun_out/ncu_a2.txt 2>&1
tail -1 gpurun_out/ncu_a2.txt
