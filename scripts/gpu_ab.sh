#!/bin/bash
# A/B bench of kernel variants in ONE GPU session (same box, same clocks regime).
# env: TAG, VARIANTS = space-separated "name:ENV=VAL,ENV2=VAL2" (name "base" = defaults),
#      BENCH_ARGS, PYTEST_ENV (env assignments for an extra pytest -m gpu pass), REPS
tag=${TAG:-ab}
out=gpurun_out/$tag
mkdir -p $out
python -c "import __graft_entry__ as g; g.build()" > $out/build.log 2>&1 || { echo BUILD FAILED; tail -30 $out/build.log; exit 1; }
if [ -n "$PYTEST_ENV" ]; then
  env $PYTEST_ENV timeout 1500 python -m pytest tests -m gpu -x -q ${PYTEST_ARGS} > $out/pytest_gpu_env.log 2>&1; echo "pytest ($PYTEST_ENV) rc=$?"
  tail -3 $out/pytest_gpu_env.log
fi
for rep in $(seq 1 ${REPS:-1}); do
for v in ${VARIANTS:-base}; do
  name=${v%%:*}; envs=""
  [ "$name" != "$v" ] && envs=$(echo ${v#*:} | tr ',' ' ')
  env $envs timeout 600 python bench.py ${BENCH_ARGS} --no-e2e --no-cpu-baseline > $out/bench_${name}_$rep.json 2>> $out/bench.err
  python -c "import json;d=json.load(open('$out/bench_${name}_$rep.json'));r=d['roofline'];print('$name rep$rep', round(d['ms_per_step'],2),'ms/step kernel frac',r['frac'],'step frac',r['step_frac_of_roofline'],'sm_mhz',d['clocks']['sm_mhz'])" || tail -5 $out/bench.err
done
done
