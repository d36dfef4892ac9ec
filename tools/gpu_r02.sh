# Round-2 evidence run on one B200: GPU tests, C4 / C1 bench lines (with
# --verify), the reference arm, and the per-kernel ncu DRAM traffic at C4.
set -x
mkdir -p gpurun_out
free -g | head -2
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -5 > gpurun_out/gpu_tests.txt
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_c4.jsonl 2> gpurun_out/bench_c4.err
timeout 600 python bench.py --config c1 --steps 50 --warmup 5 > gpurun_out/bench_c1.jsonl 2> gpurun_out/bench_c1.err
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/bench_ref.jsonl 2> gpurun_out/bench_ref.err
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
  --clock-control none -k regex:"lfps_(gate|stats|select|finish|update)_kernel" -c 60 --csv --log-file gpurun_out/launches_c4.csv \
  python bench.py --profile-only --steps 3 --warmup 3 > gpurun_out/ncu_list.log 2>&1; echo list rc $?
tail -3 gpurun_out/gpu_tests.txt
tail -c 600 gpurun_out/bench_c4.err
