# memcheck over the whole GPU suite (except the multi-process bench test)
timeout 3000 compute-sanitizer --tool memcheck --leak-check no python -m pytest tests -m gpu -q -p no:cacheprovider -k "not two_ranks and not cli" > gpurun_out/memcheck_all.txt 2>&1
grep -c "Invalid __global__\|Invalid __shared__\|out of bounds" gpurun_out/memcheck_all.txt
grep -n "passed\|failed\|ERROR SUMMARY" gpurun_out/memcheck_all.txt | tail -3
grep "Program hit" gpurun_out/memcheck_all.txt | sed 's/.*due to//' | sort | uniq -c
