# one ncu --set full capture of gemm_ex (batch $1, default 16) summarised on the box
B=${1:-16}
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:${KREGEX:-gemm_ex} -s 3 -c 1 -o /tmp/prof_ex python tools/profile_tc.py $B --exact > gpurun_out/ncu_ex.log 2>&1
tail -1 gpurun_out/ncu_ex.log
python tools/ncu_summary.py /tmp/prof_ex.ncu-rep 22052 > gpurun_out/ex_summary.txt 2>&1
python tools/ncu_srcmix.py /tmp/prof_ex.ncu-rep 22052 70 > gpurun_out/ex_srcmix.txt 2>&1
python tools/ncu_stalls.py /tmp/prof_ex.ncu-rep 40 > gpurun_out/ex_stalls.txt 2>&1
rm -f /tmp/prof_ex.ncu-rep
head -30 gpurun_out/ex_summary.txt
