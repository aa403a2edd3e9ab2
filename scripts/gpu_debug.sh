#!/bin/bash
out=gpurun_out/dbg; mkdir -p $out
python -c "import __graft_entry__ as g; g.build()" > $out/build.log 2>&1 || { echo BUILD FAILED; tail -30 $out/build.log; exit 1; }
for c in "70x37x29 cd dirichlet fp64" "70x37x29 cd dirichlet fp32" "70x37x29 2shoc msd fp64" "70x37x29 2shoc dirichlet fp64 V" \
         "70x37x29 2shoc msd fp32" "64x40x20 2shoc msd fp64" "33x18x9 2shoc l0 fp64 V"; do
  timeout 60 python scripts/debug_case.py $c 2>&1 | tail -2
done
timeout 120 compute-sanitizer --tool memcheck python scripts/debug_case.py 70x37x29 cd dirichlet fp32 2>&1 | head -40
timeout 120 compute-sanitizer --tool memcheck python scripts/debug_case.py 40x20x12 2shoc msd fp64 2>&1 | head -40
