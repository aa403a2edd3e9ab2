#!/bin/bash
# ncu --set full (+ source) of one launch of a kernel; raw csv + sass source csv. env: TAG NCU_K NCU_CFG NCU_S BARGS
tag=${TAG:-ncuf}; out=gpurun_out/$tag; mkdir -p $out
python -c "import __graft_entry__ as g; g.build()" > $out/build.log 2>&1 || { echo BUILD FAILED; exit 1; }
timeout 900 ncu --set full --import-source on --clock-control none ${NCU_EXTRA} -k regex:${NCU_K:-stage} -s ${NCU_S:-5} -c ${NCU_C:-1} \
  -o $out/prof python bench.py --config ${NCU_CFG:-trap2d} --steps 2 --warmup 1 --no-e2e --no-cpu-baseline ${BARGS} > $out/ncu.log 2>&1
echo "ncu rc=$?"
ncu -i $out/prof.ncu-rep --page raw --csv > $out/raw.csv 2>/dev/null
ncu -i $out/prof.ncu-rep --page source --csv --print-source sass > $out/sass.csv 2>/dev/null
ncu -i $out/prof.ncu-rep --page details > $out/details.txt 2>/dev/null
ls -la $out
