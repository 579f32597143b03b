# round-1 GPU pass 20: vector P2 elasticity (config 5)
set -x
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider -x 2>&1 | tail -30 > gpurun_out/pytest_gpu.txt
grep -E "passed|failed|Error|assert" gpurun_out/pytest_gpu.txt | head
