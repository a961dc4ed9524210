# batched path A/B: the batched GPU tests, then tools/batch_sweep.py with the default library and build/lib_tc0.so
python -m pytest tests/test_gpu_batched.py tests/test_gpu_fuzz.py -q -m gpu --tb=short -x 2>&1 | tail -3
python tools/batch_sweep.py --out gpurun_out/bs_new.json > /dev/null 2>&1
SPQR_LIB=$PWD/build/lib_tc0.so python tools/batch_sweep.py --out gpurun_out/bs_old.json > /dev/null 2>&1
python - <<'PY'
import json
a = json.load(open('gpurun_out/bs_old.json'))['rows']; b = json.load(open('gpurun_out/bs_new.json'))['rows']
for x, y in zip(a, b):
    print(x['batch'], 'old', x['us'], 'new', y['us'], 'cublas', y.get('cublas_fp16_us'), 'speedup_vs_cublas', y.get('speedup_vs_cublas'))
PY
