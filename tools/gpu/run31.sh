# round-1 GPU pass 31: full GPU suite incl. 2-rank bench and jitter/permutation
set -x
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider 2>&1 | tail -30 > gpurun_out/pytest_gpu.txt
grep -E "passed|failed|Error|assert" gpurun_out/pytest_gpu.txt | head
