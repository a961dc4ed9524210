# usage: TAG=... KREGEX=... bash gpurun_prof2.sh  -- one ncu --set full capture of the hot kernel
KREGEX=${KREGEX:-gemv_cta}
ncu --set full --clock-control none --import-source on -k regex:$KREGEX -s 3 -c 1 -o gpurun_out/prof_$TAG python tools/profile_gemv.py ${SHAPE:-22016 8192} > gpurun_out/ncu_$TAG.log 2>&1; tail -1 gpurun_out/ncu_$TAG.log
