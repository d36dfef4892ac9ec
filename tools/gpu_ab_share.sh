# A/B of library variants at C4 and the per-rank C4 shares; VARIANTS="a b"
for cfg in ${CONFIGS:-c4 c4s4 c4s8}; do echo "== $cfg"; BENCH_ARGS="--config $cfg" bash tools/gpu_ab2.sh 2>&1 | grep -v "^+"; done
