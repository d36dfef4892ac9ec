set -x
mkdir -p gpurun_out
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_c4.jsonl 2> gpurun_out/bench_c4.err
timeout 1500 python bench.py --config c3 --steps 5 --warmup 3 > gpurun_out/bench_c3.jsonl 2> gpurun_out/bench_c3.err
tail -c 300 gpurun_out/bench_c3.err
python -c "
import json
for f in ('gpurun_out/bench_c4.jsonl','gpurun_out/bench_c3.jsonl'):
    try:
        d=json.loads(open(f).read().strip().splitlines()[-1]); print(f, d['value'], d.get('us_per_layer_step'), d.get('setup_s'), d.get('e2e',{}).get('value'))
    except Exception as e: print(f, e)
"
