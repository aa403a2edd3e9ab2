#!/bin/bash
# bench sweep over env settings: SWEEP="VAR=val VAR=val2 ..." (each a separate bench run), BENCH_ARGS
tag=${TAG:-sweep}; out=gpurun_out/$tag; mkdir -p $out
python -c "import __graft_entry__ as g; g.build()" > $out/build.log 2>&1 || { echo BUILD FAILED; tail -30 $out/build.log; exit 1; }
if [ "${PYTEST:-0}" = "1" ]; then
  timeout 900 python -m pytest tests -m gpu -x -q ${PYTEST_ARGS} > $out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 $out/pytest_gpu.log
fi
i=0
for kv in ${SWEEP}; do
  i=$((i+1))
  env ${kv//,/ } timeout 600 python bench.py --no-e2e --no-cpu-baseline ${BENCH_ARGS} > $out/b$i.json 2>> $out/bench.err
  python -c "import json;d=json.load(open('$out/b$i.json'));print('$kv', round(d['ms_per_step'],2), 'ms/step', d['roofline']['frac'], 'kernel frac', d['pct_hbm_roofline'], '% step', d['clocks']['sm_mhz'], 'MHz')" || tail -3 $out/bench.err
done
