#!/bin/bash
# One GPU verification pass: parity tests, smoke, bench line, ncu launch list + one full capture.
# Usage (from the repo root, on the GPU box): bash scripts/gpu_check.sh [tag]
tag=${1:-r01}
out=gpurun_out/$tag
mkdir -p $out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.used --format=csv > $out/nvsmi.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > $out/build.log 2>&1 || { echo BUILD FAILED; tail -30 $out/build.log; exit 1; }
timeout ${PYT_TIMEOUT:-1800} python -m pytest tests -m gpu -x -q --durations=15 > $out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $out/pytest_gpu.log
tail -5 $out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $out/smoke.log 2>&1; echo "smoke rc=$?" >> $out/smoke.log
tail -2 $out/smoke.log
timeout 900 python bench.py > $out/bench.json 2> $out/bench.err; echo "bench rc=$?"
cat $out/bench.json
[ "$NO_NCU" = "1" ] && exit 0
# launch list of the bench command (cold-cache, serialised: compare shares)
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $out/launches.csv \
  python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > $out/ncu_launch_bench.log 2>&1; echo "ncu launches rc=$?"
# one full capture of the dominant kernel (512^3 slice of the same workload: same per-point bytes)
timeout 900 ncu --set full --clock-control none --import-source on -k regex:stage3d_stream -s 4 -c 2 \
  -o $out/prof_stage3d python bench.py --config gpe3d_512 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline \
  > $out/ncu_full.log 2>&1; echo "ncu full rc=$?"
ls -la $out
