# bench per-layer A/B of gemv_cta variant libraries (build/lib_$v.so; "default" = in-tree)
for v in ${VARIANTS:-default nc8}; do
  if [ $v = default ]; then unset SPQR_LIB; else export SPQR_LIB=$PWD/build/lib_$v.so; fi
  echo "== $v"
  timeout 400 python bench.py --steps 100 --warmup 10 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['e2e']['value'], {k: v['us'] for k, v in d['per_layer'].items()}, d['parity']['max_relative_l2'])"
done
