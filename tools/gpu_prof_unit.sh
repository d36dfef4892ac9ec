# ncu: full capture of the union + unit kernels of one unit-finish C4 step
set -x
mkdir -p gpurun_out
timeout 1500 ncu --set full --clock-control none --import-source on \
  -k regex:"lfps_(union|unit)" -s 6 -c 2 -o gpurun_out/prof_unit -f \
  python bench.py --profile-only --unit-finish --steps 2 --warmup 2 --verify 0 --no-cpu > gpurun_out/ncu_full.log 2>&1; echo full rc $?
