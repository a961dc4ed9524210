# A/B: bench with the default library and with build/lib_$V.so for each V in $VARIANTS
for v in default $VARIANTS; do
  if [ $v = default ]; then unset SPQR_LIB; else export SPQR_LIB=$PWD/build/lib_$v.so; fi
  timeout 600 python bench.py --steps 200 --warmup 20 --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/bench_$v.json
  python -c "import json; d=json.load(open('gpurun_out/bench_$v.json')); print('$v', 'value', d.get('value'), 'frac', d['roofline']['frac'], {k: v['us'] for k, v in d['per_layer'].items()}, 'e2e', d['e2e']['value'])" 2>/dev/null || tail -c 600 gpurun_out/bench_$v.json
done
