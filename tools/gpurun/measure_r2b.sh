# second closing measurement pass of round 2 (after the exact batched mode): smoke, GPU tests, bench
# both arms, launch list, DRAM traffic, full ncu captures (batch 1, gemm_tc b16, gemm_ex b16), batch
# sweeps in both modes, compute-sanitizer over every path
set -x
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
python -m pytest tests -q -m gpu --tb=short 2>&1 | tail -4
timeout 900 python bench.py 2>&1 | tail -1 > gpurun_out/bench_r2.json
head -c 3000 gpurun_out/bench_r2.json; echo
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 2>&1 | tail -1 > gpurun_out/bench_ref_r2.json
head -c 800 gpurun_out/bench_ref_r2.json; echo
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_r2.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_under_ncu.log 2>&1; tail -2 gpurun_out/launches_r2.csv
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:gemv_cta -s 4 -c 4 --csv --log-file gpurun_out/traffic_r2.csv python tools/profile_block.py > gpurun_out/traffic_r2.log 2>&1
python tools/traffic_json.py gpurun_out/traffic_r2.csv gpurun_out/traffic_r2.log gpurun_out/gemv_traffic.json | head -c 600
mkdir -p /tmp/ncu_r2
ncu --set full --clock-control none --import-source on -k regex:gemv_cta -s 3 -c 1 -o /tmp/ncu_r2/gemv python tools/profile_gemv.py > gpurun_out/ncu_r2.log 2>&1; tail -1 gpurun_out/ncu_r2.log
bash tools/profile_summary.sh /tmp/ncu_r2/gemv.ncu-rep 22016 "ncu --set full --clock-control none --import-source on -k regex:gemv_cta -s 3 -c 1 python tools/profile_gemv.py (22016x8192, 3/3/3-bit, 1% outliers, batch 1; units = 22016 cells of 32x256)" > gpurun_out/r2_gemv_cta_ncu_full.txt 2>&1
ncu --set full --clock-control none --import-source on -k regex:gemm_tc -s 2 -c 1 -o /tmp/ncu_r2/tc16 python tools/profile_tc.py 16 > gpurun_out/ncu_tc16.log 2>&1; tail -1 gpurun_out/ncu_tc16.log
bash tools/profile_summary.sh /tmp/ncu_r2/tc16.ncu-rep 22016 "ncu --set full ... -k regex:gemm_tc python tools/profile_tc.py 16 (8192x22016, batch 16; units = 22016 cells)" > gpurun_out/r2_gemm_tc_b16_ncu_full.txt 2>&1
ncu --set full --clock-control none --import-source on -k regex:gemm_ex -s 2 -c 1 -o /tmp/ncu_r2/ex16 python tools/profile_tc.py 16 --exact > gpurun_out/ncu_ex16.log 2>&1; tail -1 gpurun_out/ncu_ex16.log
bash tools/profile_summary.sh /tmp/ncu_r2/ex16.ncu-rep 22016 "ncu --set full ... -k regex:gemm_ex python tools/profile_tc.py 16 --exact (8192x22016, batch 16, exact mode; units = 22016 stages of 128x64 = cells)" > gpurun_out/r2_gemm_ex_b16_ncu_full.txt 2>&1
du -sh gpurun_out
python tools/batch_sweep.py --out gpurun_out/batch_sweep_r2.json 2>&1 | tail -1 | head -c 300; echo
python tools/batch_sweep.py --exact --out gpurun_out/batch_sweep_exact_r2.json 2>&1 | tail -1 | head -c 300; echo
for tool in memcheck synccheck initcheck; do compute-sanitizer --tool $tool --error-exitcode 9 python tools/sanitize_small.py > gpurun_out/sanitize_$tool.log 2>&1; echo "$tool rc=$?"; tail -2 gpurun_out/sanitize_$tool.log; done
