timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider 2>&1 | tail -1
timeout 3000 compute-sanitizer --tool memcheck --leak-check no python -m pytest tests -m gpu -q -p no:cacheprovider -k "not two_ranks and not cli" > gpurun_out/memcheck_all.txt 2>&1
grep -n "passed\|failed\|ERROR SUMMARY" gpurun_out/memcheck_all.txt | tail -2
