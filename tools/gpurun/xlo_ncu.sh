# ncu --set full of gemv_cta with fp16 x and fp32 x (22016x8192): where the fp32-x cost goes
mkdir -p /tmp/ncu_x gpurun_out
for dt in f16 f32; do
  ncu --set full --clock-control none --import-source on -k regex:gemv_cta -s 3 -c 1 -o /tmp/ncu_x/$dt python tools/profile_gemv.py 22016 8192 0.01 $dt > gpurun_out/ncu_x_$dt.log 2>&1
  bash tools/profile_summary.sh /tmp/ncu_x/$dt.ncu-rep 22016 "gemv_cta 22016x8192 batch 1, $dt x" > gpurun_out/xlo_$dt.txt 2>&1
  head -30 gpurun_out/xlo_$dt.txt
done
