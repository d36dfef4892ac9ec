# index-ahead prefetch: parity tests, then C3 with and without the prefetch schedule
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q --timeout 300 -k "prefetch or split or graph or host" > gpurun_out/pytest_prefetch.log 2>&1; echo pytest rc $?; tail -3 gpurun_out/pytest_prefetch.log
for v in "" "--prefetch"; do
  timeout 1500 python bench.py --config c3 --steps 5 --warmup 3 $v > gpurun_out/c3$v.jsonl 2> gpurun_out/c3$v.err
  tail -1 gpurun_out/c3$v.jsonl | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c3 $v', round(d['value'],1), round(d['us_per_layer_step'],1))"
done
