# ncu --set full of one launch each of the C4 decode kernels (profile mode: one launch per kernel per step)
set -x
mkdir -p gpurun_out
timeout 1500 ncu --set full --clock-control none --import-source on \
  -k regex:"lfps_(gate|stats|select|finish|update)_kernel" -s 10 -c 5 -o gpurun_out/prof_chain -f \
  python bench.py --profile-only --steps 2 --warmup 2 --verify 0 --no-cpu --no-split > gpurun_out/ncu_chain.log 2>&1; echo full rc $?
