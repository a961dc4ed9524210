# third closing measurement pass of round 2 (after the gemm_tc issue-block change): smoke, GPU tests,
# bench both arms, launch list, gemm_tc b16 ncu capture, batch sweep, fuzz, sanitizer
set -x
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
python -m pytest tests -q -m gpu --tb=short 2>&1 | tail -4
timeout 900 python bench.py 2>&1 | tail -1 > gpurun_out/bench_r2c.json
head -c 3000 gpurun_out/bench_r2c.json; echo
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 2>&1 | tail -1 > gpurun_out/bench_ref_r2c.json
head -c 800 gpurun_out/bench_ref_r2c.json; echo
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_r2c.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_under_ncu.log 2>&1; tail -2 gpurun_out/launches_r2c.csv
mkdir -p /tmp/ncu_r2
ncu --set full --clock-control none --import-source on -k regex:gemm_tc -s 2 -c 1 -o /tmp/ncu_r2/tc16 python tools/profile_tc.py 16 > gpurun_out/ncu_tc16.log 2>&1; tail -1 gpurun_out/ncu_tc16.log
bash tools/profile_summary.sh /tmp/ncu_r2/tc16.ncu-rep 22016 "ncu --set full ... -k regex:gemm_tc python tools/profile_tc.py 16 (8192x22016, batch 16; units = 22016 cells)" > gpurun_out/r2_gemm_tc_b16_ncu_full.txt 2>&1
python tools/batch_sweep.py --out gpurun_out/batch_sweep_r2c.json 2>&1 | tail -1 | head -c 300; echo
timeout 1200 python tools/fuzz_parity.py 1000 > gpurun_out/fuzz_r2c.txt 2>&1; tail -5 gpurun_out/fuzz_r2c.txt
for tool in memcheck synccheck; do compute-sanitizer --tool $tool --error-exitcode 9 python tools/sanitize_small.py > gpurun_out/sanitize_$tool.log 2>&1; echo "$tool rc=$?"; tail -2 gpurun_out/sanitize_$tool.log; done
