# quick GPU round trip: parity tests, smoke, one bench line (no CPU leg)
set -x
mkdir -p gpurun_out
timeout 300 python -m pytest tests -m gpu -x -q --timeout 120 > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc $?
tail -30 gpurun_out/pytest_gpu.log
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke rc $?
tail -3 gpurun_out/smoke.log
timeout 400 python bench.py --no-cpu ${BENCH_ARGS:-} > gpurun_out/bench.log 2>&1; echo bench rc $?
tail -3 gpurun_out/bench.log
