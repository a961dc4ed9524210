# sharded path checks on one GPU: NCCL C-ABI tests (world 1), bench N=1, and the N=2 bench code path with both ranks on cuda:0 (gloo hook)
python -m pytest tests/test_gpu_sharded_nccl.py tests/test_gpu.py -q -m gpu --tb=short -x 2>&1 | tail -5
timeout 600 python bench.py --steps 50 --warmup 5 --no-cpu-baseline 2>&1 | tail -1 | head -c 400; echo
SPQR_BENCH_SHARE_GPU=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/share2.log 2>&1
tail -1 gpurun_out/share2.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('share2', d['value'], d['multi_gpu'], d['parity'])" || tail -30 gpurun_out/share2.log
