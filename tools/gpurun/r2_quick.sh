# round 2 quick loop: GPU tests (-x), short bench
python -m pytest tests -q -m gpu --tb=short -x 2>&1 | tail -15
timeout 900 python bench.py --steps 200 --warmup 20 --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/bench_q.json
python -c "import json; d=json.load(open('gpurun_out/bench_q.json')); print('value', d.get('value'), 'ms/step', d.get('ms_per_step'), 'roof', d['roofline']['achieved'], d['roofline']['frac'], {k: v['us'] for k, v in d['per_layer'].items()}, 'dense', d['dense_fp16']['speedup_spqr_vs_best_dense'], 'e2e', d['e2e']['value'], 'parity', d['parity']['max_relative_l2'])" || head -c 3000 gpurun_out/bench_q.json
