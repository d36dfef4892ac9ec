# full round-end style run: tests, smoke, default bench (with the CPU leg),
# the reference arm, launch list and one ncu --set full of the hot kernels
set -x
mkdir -p gpurun_out
nproc; lscpu | grep -E "Model name|Socket|Core"
timeout 300 python -m pytest tests -m gpu -x -q --timeout 120 > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc $?
tail -3 gpurun_out/pytest_gpu.log
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke rc $?
timeout 900 python bench.py > gpurun_out/bench_full.log 2>&1; echo bench rc $?
tail -2 gpurun_out/bench_full.log
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.log 2>&1; echo ref rc $?
tail -2 gpurun_out/bench_ref.log
