# per-unit finish: parity, then C4 / C1 bench lines (unit vs session finish)
mkdir -p gpurun_out/unit
timeout 900 python -m pytest tests -m gpu -x -q -k "unit_finish or gqa or c4_context or c1_shape or golden or split or graph or block_table or paged or threads" > gpurun_out/unit/tests.txt 2>&1; echo "tests rc $?"; tail -5 gpurun_out/unit/tests.txt
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu > gpurun_out/unit/c4.jsonl 2> gpurun_out/unit/c4.err; echo "c4 rc $?"
timeout 300 python bench.py --config c1 --steps 50 --warmup 5 --no-cpu > gpurun_out/unit/c1.jsonl 2> gpurun_out/unit/c1.err; echo "c1 rc $?"
python - <<'PY'
import json
for f in ["c4", "c1"]:
    for l in open(f"gpurun_out/unit/{f}.jsonl"):
        if l.startswith("{"):
            d = json.loads(l)
            print(f, d["value"], d.get("kernel_ms"), d.get("roofline", {}).get("frac"), d.get("e2e", {}).get("value"))
PY
tail -5 gpurun_out/unit/c4.err
