# fp32-x / batch-pair kernels with shared x panels: parity tests, per-layer times, bench e2e
timeout 600 python -m pytest tests -x -q -m gpu 2>&1 | tail -2
timeout 200 python tools/xlo_cost.py 2>&1 | tail -4
timeout 300 python tools/batch_sweep.py --batches 1,2,4 2>&1 | grep "^{'"
timeout 400 python bench.py --steps 50 --warmup 10 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['e2e'])"
