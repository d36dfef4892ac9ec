# per-unit finish: parity tests, bench lines (kernel_ms) per slice count and the per-session finish, ncu of union + unit
mkdir -p gpurun_out
timeout 400 python -m pytest tests -m gpu -x -q --timeout 200 -k "unit" > gpurun_out/pytest_unit.log 2>&1; echo pytest rc $?
tail -3 gpurun_out/pytest_unit.log
run() {  # name, bench args, env...
  name=$1; shift; args=$1; shift
  env "$@" timeout 300 python bench.py --no-cpu $args --steps 10 --verify 1 --recall-steps 0 > gpurun_out/ab_$name.log 2>&1
  tail -1 gpurun_out/ab_$name.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$name', round(d['value'],1), {k: round(v*1000,1) for k,v in d['kernel_ms'].items()}, d.get('verified_units',{}).get('output_rel_err_max'))"
}
run unit "--unit-finish"
run unit_sl4 "--unit-finish" LFPS_UNIT_SLICES=4
run unit_sl1 "--unit-finish" LFPS_UNIT_SLICES=1
run session ""
for v in ${VARIANTS:-}; do run $v "--unit-finish" LFPS_LIB=$PWD/paper_2506_15704_b200/lib/variants/$v.so; done
timeout 900 ncu --set full --clock-control none --import-source on \
  -k regex:"lfps_(union|unit)" -s 6 -c 2 -o gpurun_out/prof_unit -f \
  python bench.py --profile-only --unit-finish --steps 2 --warmup 2 --verify 0 --no-cpu > gpurun_out/ncu_full.log 2>&1; echo full rc $?
