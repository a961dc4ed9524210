# closing measurement pass of a round (run under gpurun from the repo root): smoke, GPU tests,
# bench both arms, launch list, DRAM traffic per launch, full ncu captures of the batch-1 and
# batched kernels, batch and config sweeps
set -x
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
python -m pytest tests -q -m gpu --tb=short 2>&1 | tail -4
timeout 900 python bench.py 2>&1 | tail -1 > gpurun_out/bench_r1c.json
head -c 3000 gpurun_out/bench_r1c.json; echo
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 2>&1 | tail -1 > gpurun_out/bench_ref_r1c.json
head -c 600 gpurun_out/bench_ref_r1c.json; echo
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_r1c.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_under_ncu.log 2>&1; tail -2 gpurun_out/launches_r1c.csv
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:gemv_cta -s 4 -c 4 --csv --log-file gpurun_out/traffic_r1c.csv python tools/profile_block.py > gpurun_out/traffic_r1c.log 2>&1
python tools/traffic_json.py gpurun_out/traffic_r1c.csv gpurun_out/traffic_r1c.log gpurun_out/gemv_traffic.json | head -c 600
ncu --set full --clock-control none --import-source on -k regex:gemv_cta -s 3 -c 1 -o gpurun_out/prof_gemv_r1c python tools/profile_gemv.py > gpurun_out/ncu_r1c.log 2>&1; tail -1 gpurun_out/ncu_r1c.log
ncu --set full --clock-control none --import-source on -k regex:gemm_tc -s 2 -c 1 -o gpurun_out/prof_tc_r1c_b16 python tools/profile_tc.py 16 > gpurun_out/ncu_tc16.log 2>&1; tail -1 gpurun_out/ncu_tc16.log
ncu --set full --clock-control none --import-source on -k regex:gemm_tc -s 2 -c 1 -o gpurun_out/prof_tc_r1c_b64 python tools/profile_tc.py 64 > gpurun_out/ncu_tc64.log 2>&1; tail -1 gpurun_out/ncu_tc64.log
python tools/batch_sweep.py 2>&1 | tail -1 > gpurun_out/batch_sweep_r1c.json
python tools/config_sweep.py 2>&1 | tail -1 > gpurun_out/config_sweep_r1c.json
head -c 300 gpurun_out/config_sweep_r1c.json
