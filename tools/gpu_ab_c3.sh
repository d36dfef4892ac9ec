# C3 (32 layers) A/B of library variants: default first; VARIANTS="a b"
for rep in 1 2; do
for v in default ${VARIANTS:-}; do
  if [ $v = default ]; then lib=""; else lib="LFPS_LIB=$PWD/paper_2506_15704_b200/lib/variants/$v.so"; fi
  env $lib timeout 900 python bench.py --config c3 --steps 5 --warmup 3 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', round(d['value'],1), round(d['us_per_layer_step'],1))"
done; done
