set -x
timeout 300 python -m pytest tests -m gpu -x -q --timeout 120 > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc $?
tail -2 gpurun_out/pytest_gpu.log
timeout 900 python bench.py --config c3 --steps 20 --warmup 3 > gpurun_out/bench_c3.log 2>&1; echo c3 rc $?
tail -2 gpurun_out/bench_c3.log
LFPS_DIST_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --config c2 --steps 10 --warmup 3 --recall-steps 1 > gpurun_out/bench_2rank.log 2>&1; echo 2rank rc $?
tail -3 gpurun_out/bench_2rank.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29534 bench.py --impl reference --gpus 2 --config c2 --steps 2 --warmup 1 > gpurun_out/bench_2rank_ref.log 2>&1; echo 2rank ref rc $?
tail -2 gpurun_out/bench_2rank_ref.log
