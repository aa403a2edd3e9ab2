out=gpurun_out/probe1; mkdir -p $out
python -c "import __graft_entry__ as g; g.build()" > $out/build.log 2>&1
summ() { python -c "import json,sys;d=json.load(open('$1'));print('$2', round(d['ms_per_step']*1000,1),'us/step', {k:(round(v['ms']/v['launches']*1000,1),v['launches']) for k,v in d['kernel_timing'].items()})"; }
for cfg in ring3d ring3d_fp32 trap2d; do
  timeout 300 python bench.py --config $cfg --steps 336 --warmup 16 --no-e2e --no-cpu-baseline > $out/$cfg.json 2>>$out/err.log; summ $out/$cfg.json $cfg
done
for zc in 7 13 26 51; do
  NLSE_ZCHUNK=$zc timeout 300 python bench.py --config ring3d --steps 336 --warmup 16 --no-e2e --no-cpu-baseline > $out/ring_zc$zc.json 2>>$out/err.log; summ $out/ring_zc$zc.json ring3d_zc$zc
done
NLSE_TMA_TY=8 timeout 300 python bench.py --config ring3d --steps 336 --warmup 16 --no-e2e --no-cpu-baseline > $out/ring_ty8.json 2>>$out/err.log; summ $out/ring_ty8.json ring3d_ty8
timeout 300 python bench.py --config gpe3d_512 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > $out/g512.json 2>>$out/err.log; summ $out/g512.json gpe512
NLSE_FORCE_EDGE=1 timeout 300 python bench.py --config gpe3d_512 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > $out/g512fe.json 2>>$out/err.log; summ $out/g512fe.json gpe512_force_edge
tail -3 $out/err.log
