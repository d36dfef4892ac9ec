# ncu --set full of one exact-path step (score + top-k kernels) at C4
mkdir -p gpurun_out/px
timeout 1200 ncu --set full --clock-control none --import-source on \
  -k regex:"exact_(topk|score|attend)" -c 3 -o gpurun_out/px/prof_exact -f \
  python bench.py --no-cpu --verify 0 --steps 2 --warmup 3 --recall-steps 1 > gpurun_out/px/ncu.log 2>&1; echo "ncu rc $?"
python tools/ncu_summary.py gpurun_out/px/prof_exact.ncu-rep
