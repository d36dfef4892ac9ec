set -x
timeout 300 python bench.py --no-cpu --steps 100 --recall-steps 1 > gpurun_out/b_base.log 2>&1; echo rc $?
timeout 300 python bench.py --no-cpu --steps 100 --recall-steps 1 --split > gpurun_out/b_split.log 2>&1; echo rc $?
