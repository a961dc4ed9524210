# one ncu --set full capture of gemm_tc (batch $1, default 16) summarised on the box
B=${1:-16}
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_tc -s 3 -c 1 -o /tmp/prof_tc python tools/profile_tc.py $B > gpurun_out/ncu_tc.log 2>&1
tail -1 gpurun_out/ncu_tc.log
python tools/ncu_srcmix.py /tmp/prof_tc.ncu-rep 22016 80 > gpurun_out/tc_srcmix.txt 2>&1
python tools/ncu_stalls.py /tmp/prof_tc.ncu-rep 40 > gpurun_out/tc_stalls.txt 2>&1
rm -f /tmp/prof_tc.ncu-rep
