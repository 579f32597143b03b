timeout 2400 compute-sanitizer --tool racecheck python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider \
  -k "elasticity_class or (gpu_matches_oracle and gather) or isolated or window" > gpurun_out/racecheck2.txt 2>&1
grep -n "hazard\|RACECHECK SUMMARY\|passed\|failed" gpurun_out/racecheck2.txt | tail -5
timeout 1200 compute-sanitizer --tool synccheck python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider \
  -k "class_specialised or elasticity_class" > gpurun_out/synccheck.txt 2>&1
grep -n "ERROR SUMMARY\|passed\|failed" gpurun_out/synccheck.txt | tail -3
