# exact path: parity tests, then the C4 exact-path timing (bench recall leg) and ncu
mkdir -p gpurun_out/px
timeout 600 python -m pytest tests -m gpu -x -q -k "exact or golden or gqa" > gpurun_out/px/tests.txt 2>&1; echo "tests rc $?"; tail -2 gpurun_out/px/tests.txt
timeout 600 python bench.py --no-cpu --verify 0 --steps 10 --warmup 3 --recall-steps 3 > gpurun_out/px/c4.jsonl 2>gpurun_out/px/c4.err; echo "bench rc $?"
python -c "
import json
for l in open('gpurun_out/px/c4.jsonl'):
    if l.startswith('{'):
        d=json.loads(l); r=d['recall']; print('exact', r['exact_us_per_step'], r['exact_kernel_ms'], 'step', d['value'])
"
bash tools/gpu_prof_exact.sh
