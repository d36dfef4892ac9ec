set -x
mkdir -p gpurun_out
timeout 300 python -m pytest tests -m gpu -x -q --timeout 120 > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc $?
tail -3 gpurun_out/pytest_gpu.log
timeout 400 python bench.py --no-cpu --steps 50 --recall-steps 1 > gpurun_out/bench.log 2>&1; echo bench rc $?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"lfps_finish" -s 2 -c 1 -o gpurun_out/prof_fin -f python bench.py --profile-only --steps 2 --warmup 2 > gpurun_out/ncu_full.log 2>&1; echo ncu rc $?
