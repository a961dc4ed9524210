for v in default nc16p nc20 nc24; do
  if [ $v = default ]; then unset SPQR_LIB; else export SPQR_LIB=$PWD/build/lib_$v.so; fi
  timeout 600 python bench.py --steps 200 --warmup 20 --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/bench_$v.json
  python -c "import json; d=json.load(open('gpurun_out/bench_$v.json')); print('$v', 'value', d.get('value'), 'frac', d['roofline']['frac'], {k: v['us'] for k, v in d['per_layer'].items()}, 'e2e', d['e2e']['value'])" || tail -c 1000 gpurun_out/bench_$v.json
done
