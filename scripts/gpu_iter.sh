#!/bin/bash
# Iteration pass: build, gpu tests, bench (default kernel) + optional A/B variants, ncu of the top kernel.
# env: TAG (output dir), PYTEST_ARGS, BENCH_ARGS, AB (space-separated NLSE_3D_KERNEL values), NCU=0/1, NCU_CFG
tag=${TAG:-iter}
out=gpurun_out/$tag
mkdir -p $out
python -c "import __graft_entry__ as g; g.build()" > $out/build.log 2>&1 || { echo BUILD FAILED; tail -30 $out/build.log; exit 1; }
if [ "${PYTEST:-1}" = "1" ]; then
  timeout 1500 python -m pytest tests -m gpu -x -q ${PYTEST_ARGS} > $out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
  tail -15 $out/pytest_gpu.log
fi
timeout 900 python bench.py ${BENCH_ARGS} > $out/bench.json 2> $out/bench.err; echo "bench rc=$?"; cat $out/bench.json; tail -3 $out/bench.err
for v in ${AB}; do
  NLSE_3D_KERNEL=$v timeout 900 python bench.py ${BENCH_ARGS} --no-e2e --no-cpu-baseline > $out/bench_$v.json 2>> $out/bench.err
  echo "AB $v:"; python -c "import json;d=json.load(open('$out/bench_$v.json'));print(d['value'],d['ms_per_step'],d['roofline']['frac'],d['kernel_timing'])"
done
if [ "${NCU:-0}" = "1" ]; then
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $out/launches.csv \
    python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline ${BENCH_ARGS} > $out/ncu_launch.log 2>&1; echo "ncu launches rc=$?"
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:${NCU_K:-stage3d} -s ${NCU_S:-8} -c ${NCU_C:-4} \
    -o $out/prof python bench.py --config ${NCU_CFG:-gpe3d_512} --steps 2 --warmup 1 --no-e2e --no-cpu-baseline \
    > $out/ncu_full.log 2>&1; echo "ncu full rc=$?"
fi
ls $out
