FF_G2=1 timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "gather or class or isolated" -p no:cacheprovider 2>&1 | tail -1 > gpurun_out/t80.txt
for c in ns c3 c2; do for v in FF_NONE=1 FF_G2=1 "FF_G2=1 FF_EINV_L1=1"; do
  echo "$c $v $(env $v timeout 300 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 0 2>/dev/null | python -c "import json,sys;d=json.load(sys.stdin);print(round(d['ms_per_step'],4), round(d['config'].get('k2a_ms'),4), round(d['config'].get('k2_ms'),4))")"
done; done
cat gpurun_out/t80.txt
