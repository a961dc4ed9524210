# round-1 measurement pass for the current kernel: tests, bench line, launch list,
# DRAM traffic per launch, one full ncu capture of the hot kernel
set -x
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
python -m pytest tests -q -m gpu --tb=short 2>&1 | tail -4
timeout 900 python bench.py 2>&1 | tail -1 > gpurun_out/bench_r1b.json
head -c 3000 gpurun_out/bench_r1b.json; echo
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_r1b.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_under_ncu.log 2>&1; tail -2 gpurun_out/launches_r1b.csv
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:gemv_cta -s 4 -c 4 --csv --log-file gpurun_out/traffic_r1b.csv python tools/profile_block.py > gpurun_out/traffic_r1b.log 2>&1
python tools/traffic_json.py gpurun_out/traffic_r1b.csv gpurun_out/traffic_r1b.log gpurun_out/gemv_traffic.json | head -c 600
ncu --set full --clock-control none --import-source on -k regex:gemv_cta -s 3 -c 1 -o gpurun_out/prof_gemv_r1b python tools/profile_gemv.py > gpurun_out/ncu_r1b.log 2>&1; tail -1 gpurun_out/ncu_r1b.log
