# compute-sanitizer memcheck over the gather paths (small meshes)
timeout 1500 compute-sanitizer --tool memcheck --leak-check no python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider \
  -k "isolated or (elasticity_matches and gather) or class_specialised or gather_plan_covers or jittered" > gpurun_out/memcheck.txt 2>&1
grep -n "=========.*Invalid\|=========     at\|Address\|ERROR SUMMARY\|is out of bounds\|Program hit" gpurun_out/memcheck.txt | head -40
