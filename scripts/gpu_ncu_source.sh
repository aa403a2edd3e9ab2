#!/bin/bash
# One stage kernel with SourceCounters only (small report): per-instruction executed counts + stalls.
tag=${TAG:-ncus}; out=gpurun_out/$tag; mkdir -p $out
python -c "import __graft_entry__ as g; g.build()" > $out/build.log 2>&1 || { echo BUILD FAILED; exit 1; }
timeout 900 ncu --section SourceCounters --section WarpStateStats --clock-control none -k regex:${NCU_K:-stage3d} -s ${NCU_S:-5} -c 1 \
  -o $out/src python bench.py --config ${NCU_CFG:-gpe3d_256} --steps 2 --warmup 1 --no-e2e --no-cpu-baseline ${BENCH_ARGS} > $out/ncu.log 2>&1
echo "ncu rc=$?"; ls -la $out
ncu -i $out/src.ncu-rep --page source --csv --print-source sass > $out/sass.csv 2>/dev/null
rm -f $out/src.ncu-rep
ls -la $out
