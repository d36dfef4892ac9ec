# A/B of library variants: C4 bench lines (kernel_ms), default build first; VARIANTS="a b"
mkdir -p gpurun_out
run() {  # name, env...
  name=$1; shift
  env "$@" timeout 300 python bench.py --no-cpu ${BENCH_ARGS:-} --steps 20 --verify 1 --recall-steps 0 > gpurun_out/ab_$name.log 2>&1
  tail -1 gpurun_out/ab_$name.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$name', round(d['value'],1), {k: round(v*1000,1) for k,v in d['kernel_ms'].items()}, 'e2e', round(d['e2e']['value'],1))"
}
if [ -n "${TESTS:-}" ]; then timeout 400 python -m pytest tests -m gpu -x -q --timeout 200 -k "$TESTS" > gpurun_out/pytest_ab.log 2>&1; echo pytest rc $?; tail -2 gpurun_out/pytest_ab.log; fi
for rep in 1 2; do
run default
for v in ${VARIANTS:-}; do run $v LFPS_LIB=$PWD/paper_2506_15704_b200/lib/variants/$v.so; done
done
