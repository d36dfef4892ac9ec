# ncu evidence for the decode step at C4: launch list of our kernels, then one
# full capture of the given kernels (one launch each).
set -x
mkdir -p gpurun_out
KREGEX=${KREGEX:-lfps_(select|finish)}
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
  --clock-control none -k regex:"lfps_(clear|gate|stats|select|finish|update|append|commit)" -c 40 --csv --log-file gpurun_out/launches.csv \
  python bench.py --profile-only --steps 3 --warmup 3 > gpurun_out/ncu_list.log 2>&1; echo list rc $?
timeout 1500 ncu --set full --clock-control none --import-source on \
  -k regex:"$KREGEX" -s 4 -c 2 -o gpurun_out/prof_c4 -f \
  python bench.py --profile-only --steps 2 --warmup 2 > gpurun_out/ncu_full.log 2>&1; echo full rc $?
ls -la gpurun_out
