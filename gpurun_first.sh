python -m pytest tests -q -m gpu --tb=short 2>&1 | tail -4
timeout 600 python bench.py --steps 300 --warmup 30 --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/bench_v10.json
python -c "import json; d=json.load(open('gpurun_out/bench_v10.json')); print('value', d['value'], 'ms/step', d['ms_per_step'], 'roof', d['roofline']['achieved'], d['roofline']['frac'], {k: v['us'] for k, v in d['per_layer'].items()}, 'dense', d['dense_fp16']['speedup_spqr_vs_best_dense'])"
ncu --set full --clock-control none --import-source on -k regex:gemv_tiled -s 3 -c 1 -o gpurun_out/prof_gemv_v10 python tools/profile_gemv.py > gpurun_out/ncu_v10.log 2>&1; tail -1 gpurun_out/ncu_v10.log
