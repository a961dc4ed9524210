# last pass of the round: smoke, full GPU suite, bench (both arms)
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python -m pytest tests -q -m gpu 2>&1 | tail -2
timeout 900 python bench.py 2>&1 | tail -1 > gpurun_out/bench_final2.json
python -c "import json; d=json.load(open('gpurun_out/bench_final2.json')); print(d['value'], d['roofline']['frac'], d['e2e'], d['clocks'], d['parity']['max_relative_l2'], d['dense_fp16']['speedup_spqr_vs_best_dense'])"
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 2>&1 | tail -1 > gpurun_out/bench_ref_final2.json
head -c 300 gpurun_out/bench_ref_final2.json; echo
