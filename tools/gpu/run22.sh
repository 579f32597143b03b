# round-1 GPU pass 22: linalg consumer tests
set -x
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider 2>&1 | tail -30 > gpurun_out/pytest_gpu.txt
grep -E "passed|failed|Error|assert" gpurun_out/pytest_gpu.txt | head
