# round evidence: launch list of one decode step + exact step, full ncu of
# the decode kernels, all at C4 (one GPU, never multi-rank)
set -x
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
  --clock-control none -k regex:"lfps_(gate|stats|select|finish|update|exact)" -c 40 --csv \
  --log-file gpurun_out/launches_c4.csv python bench.py --profile-only --no-split --steps 2 --warmup 3 \
  > gpurun_out/ncu_list.log 2>&1; echo list rc $?
timeout 1500 ncu --set full --clock-control none --import-source on \
  -k regex:"lfps_(gate|stats|select|finish|update)" -s 5 -c 5 -o gpurun_out/prof_c4_full -f \
  python bench.py --profile-only --no-split --steps 2 --warmup 2 > gpurun_out/ncu_full.log 2>&1; echo full rc $?
