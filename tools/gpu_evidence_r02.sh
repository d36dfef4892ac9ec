# Round-2 evidence at HEAD on one B200: C4 (default bench line incl. the
# stock-reference cpu_baseline and --verify), C1, C2, C3, the reference arm,
# the C5 sweep, the ncu launch lists (per-kernel DRAM traffic) and one ncu
# --set full capture of the five decode kernels at C4.
set -x
mkdir -p gpurun_out/ev
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/ev/c4.jsonl 2> gpurun_out/ev/c4.err
timeout 600 python bench.py --config c1 --steps 50 --warmup 5 > gpurun_out/ev/c1.jsonl 2> gpurun_out/ev/c1.err
timeout 600 python bench.py --config c2 --steps 50 --warmup 5 > gpurun_out/ev/c2.jsonl 2> gpurun_out/ev/c2.err
timeout 1500 python bench.py --config c3 --steps 5 --warmup 3 > gpurun_out/ev/c3.jsonl 2> gpurun_out/ev/c3.err
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/ev/ref.jsonl 2> gpurun_out/ev/ref.err
timeout 1500 python tools/sweep.py --out gpurun_out/ev/sweep.jsonl > gpurun_out/ev/sweep.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
  --clock-control none -k regex:"lfps_(gate|stats|select|finish|update)_kernel" -s 45 -c 45 --csv --log-file gpurun_out/ev/launches_c4.csv \
  python bench.py --profile-only --steps 3 --warmup 3 > gpurun_out/ev/ncu_list.log 2>&1; echo list rc $?
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
  --clock-control none -k regex:"lfps_(gate|stats|select|finish|update)_kernel" -s 25 -c 25 --csv --log-file gpurun_out/ev/launches_c1.csv \
  python bench.py --config c1 --profile-only --steps 3 --warmup 3 > gpurun_out/ev/ncu_list_c1.log 2>&1; echo list rc $?
timeout 1500 ncu --set full --clock-control none --import-source on \
  -k regex:"lfps_(gate|stats|select|finish|update)_kernel" -s 10 -c 5 -o gpurun_out/ev/prof_c4 -f \
  python bench.py --profile-only --steps 2 --warmup 2 --verify 0 --no-cpu --no-split > gpurun_out/ev/ncu_full.log 2>&1; echo full rc $?
for f in c4 c1 c2 c3 ref; do tail -c 300 gpurun_out/ev/$f.err; done
