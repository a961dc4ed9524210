python -m pytest tests -q -m gpu --tb=short -x 2>&1 | tail -4
timeout 600 python bench.py --steps 300 --warmup 30 --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/bench_q.json
python -c "import json; d=json.load(open('gpurun_out/bench_q.json')); print('value', d['value'], 'ms/step', d['ms_per_step'], 'roof', d['roofline']['achieved'], d['roofline']['frac'], {k: v['us'] for k, v in d['per_layer'].items()}, 'dense', d['dense_fp16']['speedup_spqr_vs_best_dense'], 'e2e', d['e2e']['value'])"
