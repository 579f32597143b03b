timeout 600 ncu --set full --clock-control none --import-source on -k regex:ff_gather_classes -s 1 -c 1 -o gpurun_out/prof_ns_r48 \
  python bench.py --steps 2 --warmup 1 --e2e-steps 0 --no-cpu-baseline > gpurun_out/ncu_r48.txt 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_ns_gather.csv \
  python bench.py --steps 2 --warmup 1 --e2e-steps 0 --no-cpu-baseline > gpurun_out/ncu_launch_bench.txt 2>&1
tail -1 gpurun_out/ncu_r48.txt
