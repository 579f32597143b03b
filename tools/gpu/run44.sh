FF_IPW=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:ff_gather_classes -s 1 -c 1 -o gpurun_out/prof_c5cls2 \
  python bench.py --config c5 --steps 1 --warmup 1 --e2e-steps 0 --no-cpu-baseline > gpurun_out/ncu_c5.txt 2>&1
tail -1 gpurun_out/ncu_c5.txt
