# ncu --set full of gemm_tc at batch 16 (8192x22016), summarised on the box
mkdir -p /tmp/ncu_r2 gpurun_out
ncu --set full --clock-control none --import-source on -k regex:gemm_tc -s 2 -c 1 -o /tmp/ncu_r2/tc16 python tools/profile_tc.py 16 > gpurun_out/ncu_tc16.log 2>&1; tail -1 gpurun_out/ncu_tc16.log
bash tools/profile_summary.sh /tmp/ncu_r2/tc16.ncu-rep 22016 "ncu --set full ... -k regex:gemm_tc python tools/profile_tc.py 16 (8192x22016, batch 16: 9-warp layout, 2 column halves per dequant warp; units = 22016 cells)" > gpurun_out/r2_gemm_tc_b16_ncu_full.txt 2>&1
head -14 gpurun_out/r2_gemm_tc_b16_ncu_full.txt
