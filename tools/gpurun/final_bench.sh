# final bench lines of the round (both arms) + launch list, after the host-path and fp32-panel changes
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py 2>&1 | tail -1 > gpurun_out/bench_final.json
python -c "import json; d=json.load(open('gpurun_out/bench_final.json')); print(d['value'], d['roofline']['frac'], d['e2e'], d['clocks'], d['parity']['max_relative_l2'])"
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 2>&1 | tail -1 > gpurun_out/bench_ref_final.json
head -c 600 gpurun_out/bench_ref_final.json; echo
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_final.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_under_ncu.log 2>&1; tail -2 gpurun_out/launches_final.csv
