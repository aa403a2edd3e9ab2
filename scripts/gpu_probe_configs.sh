#!/bin/bash
# Per-kernel timing of the small BASELINE configurations (bench.py --config ...), one line each.
out=gpurun_out/${TAG:-probe}; mkdir -p $out
python -c "import __graft_entry__ as g; g.build()" > $out/build.log 2>&1
summ() { python -c "import json,sys;d=json.load(open('$1'));print('$2', round(d['ms_per_step']*1000,1),'us/step', {k:(round(v['ms']/v['launches']*1000,1),v['launches']) for k,v in d['kernel_timing'].items()})"; }
for cfg in ${CFGS:-ring3d ring3d_fp32 trap2d}; do
  timeout 300 python bench.py --config $cfg --steps 336 --warmup 16 --no-e2e --no-cpu-baseline > $out/$cfg.json 2>>$out/err.log; summ $out/$cfg.json $cfg
done
