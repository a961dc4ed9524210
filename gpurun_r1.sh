set -x
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
python -m pytest tests -q -m gpu --tb=short 2>&1 | tail -4
timeout 900 python bench.py 2>&1 | tail -1 > gpurun_out/bench_r1.json
cat gpurun_out/bench_r1.json | head -c 3000; echo
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_r1.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_under_ncu.log 2>&1; tail -2 gpurun_out/launches_r1.csv
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:gemv_tiled -s 7 -c 7 --csv --log-file gpurun_out/traffic_r1.csv python tools/profile_block.py > gpurun_out/traffic_r1.log 2>&1
python tools/traffic_json.py gpurun_out/traffic_r1.csv gpurun_out/traffic_r1.log gpurun_out/gemv_traffic.json | head -c 600
ncu --set full --clock-control none --import-source on -k regex:gemv_tiled -s 3 -c 1 -o gpurun_out/prof_gemv_r1 python tools/profile_gemv.py > gpurun_out/ncu_r1.log 2>&1; tail -1 gpurun_out/ncu_r1.log
