timeout 1500 compute-sanitizer --tool memcheck --leak-check no python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider \
  -k "elasticity_class or window or row_blocks_concatenate or (gpu_matches_oracle and gather)" > gpurun_out/memcheck2.txt 2>&1
grep -n "Invalid\|out of bounds\|ERROR SUMMARY\|passed\|failed" gpurun_out/memcheck2.txt | head -10
timeout 1500 compute-sanitizer --tool racecheck python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider \
  -k "class_specialised and poisson" > gpurun_out/racecheck.txt 2>&1
grep -n "hazard\|RACECHECK SUMMARY\|ERROR SUMMARY\|passed\|failed" gpurun_out/racecheck.txt | head -10
