# round 2 iteration: GPU tests (-x), short bench, one ncu --set full capture of gemv_cta (TAG=...)
TAG=${TAG:-iter}
python -m pytest tests -q -m gpu --tb=short -x ${TESTS:-} 2>&1 | tail -8
timeout 900 python bench.py --steps 200 --warmup 20 --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/bench_$TAG.json
python -c "import json; d=json.load(open('gpurun_out/bench_$TAG.json')); print('value', d.get('value'), 'ms/step', d.get('ms_per_step'), 'frac', d['roofline']['frac'], {k: v['us'] for k, v in d['per_layer'].items()}, 'e2e', d['e2e']['value'], 'parity', d['parity']['max_relative_l2'])" || tail -c 3000 gpurun_out/bench_$TAG.json
if [ -z "$NO_NCU" ]; then
ncu --set full --clock-control none --import-source on -k regex:${KREGEX:-gemv_cta} -s 3 -c 1 -o gpurun_out/prof_$TAG python tools/profile_gemv.py ${SHAPE:-22016 8192} > gpurun_out/ncu_$TAG.log 2>&1
bash tools/profile_summary.sh gpurun_out/prof_$TAG.ncu-rep ${UNITS:-22016} "$TAG gemv_cta ${SHAPE:-22016 8192}" > gpurun_out/summary_$TAG.txt 2>&1
head -40 gpurun_out/summary_$TAG.txt
fi
