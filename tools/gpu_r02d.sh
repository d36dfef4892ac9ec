set -x
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_reference_suite.py tests/test_gpu_lfps_api.py -q 2>&1 | tail -8 > gpurun_out/ref_suite2.txt
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
  --clock-control none -k regex:"lfps_(gate|stats|select|finish|update)_kernel" -s 45 -c 45 --csv --log-file gpurun_out/launches_c4.csv \
  python bench.py --profile-only --steps 3 --warmup 3 > gpurun_out/ncu_list.log 2>&1; echo list rc $?
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
  --clock-control none -k regex:"lfps_(gate|stats|select|finish|update)_kernel" -s 25 -c 25 --csv --log-file gpurun_out/launches_c1.csv \
  python bench.py --config c1 --profile-only --steps 3 --warmup 3 > gpurun_out/ncu_list_c1.log 2>&1; echo list rc $?
timeout 1500 ncu --set full --clock-control none --import-source on \
  -k regex:"lfps_(stats|select|finish|update)_kernel" -s 12 -c 4 -o gpurun_out/r02_c4_full -f \
  python bench.py --profile-only --steps 2 --warmup 3 --no-split > gpurun_out/ncu_full.log 2>&1; echo full rc $?
cat gpurun_out/ref_suite2.txt
