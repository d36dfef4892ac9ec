# per-unit finish: parity tests, then C4 bench lines (per-session vs unit)
set -x
mkdir -p gpurun_out
timeout 400 python -m pytest tests -m gpu -x -q --timeout 200 -k "unit" > gpurun_out/pytest_unit.log 2>&1; echo pytest rc $?
tail -15 gpurun_out/pytest_unit.log
timeout 300 python bench.py --no-cpu --unit-finish --steps 20 --verify 2 > gpurun_out/bench_unit.log 2>&1; echo bench rc $?
tail -c 400 gpurun_out/bench_unit.log
