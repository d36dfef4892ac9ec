# parity tests on the default build, then A/B over configs
timeout 600 python -m pytest tests -m gpu -x -q --timeout 200 > gpurun_out/pytest_front.log 2>&1; echo pytest rc $?; tail -3 gpurun_out/pytest_front.log
for cfg in ${CONFIGS:-c4 c4s4 c4s8 c1 c2}; do echo "== $cfg"; BENCH_ARGS="--config $cfg" bash tools/gpu_ab2.sh 2>&1 | grep -v "^+"; done
