#!/bin/bash
# A/B over configs x variants in one session. env: TAG, CFGS, VARIANTS ("name:ENV=V,ENV2=V"), STEPS, REPS
out=gpurun_out/${TAG:-ab2}; mkdir -p $out
python -c "import __graft_entry__ as g; g.build()" > $out/build.log 2>&1 || { echo BUILD FAILED; tail -30 $out/build.log; exit 1; }
if [ -n "$PYT" ]; then timeout 1200 python -m pytest -x -q $PYT > $out/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 $out/pytest.log; fi
for rep in $(seq 1 ${REPS:-1}); do
for cfg in ${CFGS:-trap2d}; do
for v in ${VARIANTS:-base}; do
  name=${v%%:*}; envs=""
  [ "$name" != "$v" ] && envs=$(echo ${v#*:} | tr ',' ' ')
  f=$out/${cfg}_${name}_$rep.json
  env $envs timeout 300 python bench.py --config $cfg --steps ${STEPS:-200} --warmup 20 --no-e2e --no-cpu-baseline $BARGS > $f 2>> $out/bench.err
  python -c "import json;d=json.load(open('$f'));r=d['roofline'];print('$cfg $name r$rep', round(d['ms_per_step']*1000,1),'us/step', '%.3e'%d['value'], 'kfrac',r['frac'],'sfrac',r['step_frac_of_roofline'],'mhz',d['clocks']['sm_mhz'], {k:round(v['ms']/v['launches']*1000,2) for k,v in d['kernel_timing'].items()})" || tail -3 $out/bench.err
done; done; done
