# the per-rank shares of C4 at 2 / 4 / 8 GPUs, measured on one GPU
mkdir -p gpurun_out
for cfg in c4s2 c4s4 c4s8; do
  timeout 300 python bench.py --config $cfg --no-cpu --steps 30 --recall-steps 0 --verify 1 > gpurun_out/sh_$cfg.log 2>&1
  tail -1 gpurun_out/sh_$cfg.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$cfg', round(d['value'],1), {k: round(v*1000,1) for k,v in d['kernel_ms'].items()}, 'e2e', round(d['e2e']['value'],1), 'phase', {k: round(v,1) for k,v in d['phase_us']['finish'].items()})"
done
