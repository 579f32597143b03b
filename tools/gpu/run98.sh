timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "class_specialised" -p no:cacheprovider 2>&1 | tail -1 > gpurun_out/t98.txt
FF_CWARPS=2 FF_MINB_S=6 timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "class_specialised" -p no:cacheprovider 2>&1 | tail -1 >> gpurun_out/t98.txt
for v in FF_NONE=1 "FF_CWARPS=2 FF_MINB_S=6" "FF_CWARPS=1 FF_MINB_S=12" "FF_CWARPS=2 FF_MINB_S=6 FF_IPW=3"; do
  echo "ns $v $(env $v timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 0 2>/dev/null | python -c "import json,sys;d=json.load(sys.stdin);print(round(d['ms_per_step'],4))")"
done
cat gpurun_out/t98.txt
