# round-1 GPU pass 29: profile of the current default step
set -x
timeout 600 ncu --set full --clock-control none --import-source on -k regex:ff_gather_classes -s 1 -c 1 -o gpurun_out/prof_cls_final2 \
  python bench.py --steps 2 --warmup 1 --e2e-steps 0 --no-cpu-baseline > gpurun_out/ncu_full.txt 2>&1
tail -2 gpurun_out/ncu_full.txt
