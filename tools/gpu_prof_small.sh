set -x
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"lfps_(update|gate|select)" -s 6 -c 3 -o gpurun_out/prof_ug -f python bench.py --profile-only --steps 2 --warmup 3 > gpurun_out/ncu_ug.log 2>&1; echo ncu rc $?
