# parity tests on the default build, then one bench line per library variant
# (VARIANTS="s2 ..." under paper_2506_15704_b200/lib/variants/)
mkdir -p gpurun_out
timeout 300 python -m pytest tests -m gpu -x -q --timeout 120 > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc $?
tail -5 gpurun_out/pytest_gpu.log
timeout 300 python bench.py --no-cpu ${BENCH_ARGS:-} > gpurun_out/bench.log 2>&1; echo bench rc $?
tail -1 gpurun_out/bench.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('default', d['value'], d['kernel_ms'], d['e2e']['value'])"
for v in ${VARIANTS:-}; do
  if [ "$v" = nosplit ]; then
    timeout 300 python bench.py --no-cpu --no-split ${BENCH_ARGS:-} > gpurun_out/bench_$v.log 2>&1; echo bench $v rc $?
  else
    LFPS_LIB=$PWD/paper_2506_15704_b200/lib/variants/$v.so timeout 300 python bench.py --no-cpu ${BENCH_ARGS:-} > gpurun_out/bench_$v.log 2>&1; echo bench $v rc $?
  fi
  tail -1 gpurun_out/bench_$v.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', d['value'], d['kernel_ms'], d['e2e']['value'])"
done
