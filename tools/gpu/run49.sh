timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "two_ranks" -p no:cacheprovider 2>&1 | tail -3
for c in c1 c2 c5; do
FF_BENCH_SHARE_GPU=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr 127.0.0.1 --master-port 29541 bench.py --gpus 2 --config $c --size 12 --steps 3 --warmup 3 --e2e-steps 1 2>/dev/null | grep '^{' | python -c "import json,sys;d=json.load(sys.stdin);print('$c', d['scaling'], d['config']['elements'], d['config']['dofs'], d['config']['nnz'], d['value'] > 0, d['config']['workload'][-60:])"
done
