# Round-2: the new GPU tests, the multi-rank bench path on one B200 (gloo
# ranks sharing the device: correctness of the sharded path, not scaling),
# and the per-kernel ncu DRAM traffic at C4.
set -x
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_sharded.py tests/test_gpu_parity.py -q -x -k "sharded or two_threads or failed or host" 2>&1 | tail -5 > gpurun_out/gpu_tests_b.txt
LFPS_DIST_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --config c2 --steps 10 --warmup 3 --no-cpu > gpurun_out/bench_c2_2rank.jsonl 2> gpurun_out/bench_c2_2rank.err
LFPS_DIST_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus 2 --config c1 --steps 10 --warmup 3 --no-cpu > gpurun_out/bench_c1_2rank.jsonl 2> gpurun_out/bench_c1_2rank.err
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
  --clock-control none -k regex:"lfps_(gate|stats|select|finish|update)_kernel" -s 45 -c 45 --csv --log-file gpurun_out/launches_c4.csv \
  python bench.py --profile-only --steps 3 --warmup 3 > gpurun_out/ncu_list.log 2>&1; echo list rc $?
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
  --clock-control none -k regex:"lfps_(gate|stats|select|finish|update)_kernel" -s 25 -c 25 --csv --log-file gpurun_out/launches_c1.csv \
  python bench.py --config c1 --profile-only --steps 3 --warmup 3 > gpurun_out/ncu_list_c1.log 2>&1; echo list rc $?
cat gpurun_out/gpu_tests_b.txt
tail -c 400 gpurun_out/bench_c2_2rank.err gpurun_out/bench_c1_2rank.err
