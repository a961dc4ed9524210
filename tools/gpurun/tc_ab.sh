# A/B of gemm_tc library variants (build/lib_$v.so; "default" = the in-tree library)
for v in ${VARIANTS:-default}; do
  if [ $v = default ]; then unset SPQR_LIB; else export SPQR_LIB=$PWD/build/lib_$v.so; fi
  echo "== $v"
  timeout 300 python tools/batch_sweep.py --batches ${BATCHES:-8,16,32,64} 2>&1 | tail -${TAILN:-6}
done
