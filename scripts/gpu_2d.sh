#!/bin/bash
# 2D strip kernel: parity tests + trap2d bench A/B (strip vs tile)
out=gpurun_out/${TAG:-s2d}
mkdir -p $out
python -c "import __graft_entry__ as g; g.build()" > $out/build.log 2>&1 || { echo BUILD FAILED; tail -30 $out/build.log; exit 1; }
timeout 900 python -m pytest -x -q tests/test_gpu_strip2d.py "tests/test_gpu_parity.py::test_matrix_bitwise" tests/test_gpu_slabs.py tests/test_gpu_parity2.py -k "strip or 2d or matrix_bitwise" > $out/pytest.log 2>&1; echo "pytest rc=$?"; tail -15 $out/pytest.log
for cfg in ${CFGS:-trap2d trap2d_4096}; do
for v in strip tile; do
  if [ $v = tile ]; then export NLSE_2D_KERNEL=tile; else unset NLSE_2D_KERNEL; fi
  timeout 300 python bench.py --config $cfg --steps ${STEPS:-200} --warmup 20 --no-e2e --no-cpu-baseline > $out/bench_${cfg}_$v.json 2>> $out/bench.err
  python -c "import json;d=json.load(open('$out/bench_${cfg}_$v.json'));r=d['roofline'];print('$cfg $v', round(d['ms_per_step']*1000,1),'us/step', '%.3e'%d['value'], 'kernel frac',r['frac'],'step frac',r['step_frac_of_roofline'],'sm_mhz',d['clocks']['sm_mhz'], {k:round(v['ms']/v['launches']*1000,2) for k,v in d['kernel_timing'].items()})" || tail -5 $out/bench.err
done
done
