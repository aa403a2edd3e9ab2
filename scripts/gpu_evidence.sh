#!/bin/bash
# Evidence pass for profiles/: the default bench line, the ncu launch list of the same command,
# one `ncu --set full` capture of the four stage launches of one RK4 step (512^3 slice of the
# workload, same per-point bytes) summarised into dram bytes per point, and per-instruction
# source counters of one stage-2 launch.  Usage: TAG=r01x bash scripts/gpu_evidence.sh
tag=${TAG:-ev}; out=gpurun_out/$tag; mkdir -p $out
python -c "import __graft_entry__ as g; g.build()" > $out/build.log 2>&1 || { echo BUILD FAILED; exit 1; }
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,power.limit --format=csv > $out/nvsmi.txt 2>&1
timeout 900 python bench.py > $out/bench.json 2> $out/bench.err; echo "bench rc=$?"; cat $out/bench.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $out/launches.csv \
  python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > $out/ncu_launch.log 2>&1; echo "ncu launches rc=$?"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:stage3d_tma -s 8 -c 4 \
  -o $out/full python bench.py --config gpe3d_512 --steps 2 --warmup 1 --no-e2e --no-cpu-baseline \
  > $out/ncu_full.log 2>&1; echo "ncu full rc=$?"
ncu -i $out/full.ncu-rep --page raw --csv > $out/full_raw.csv 2>/dev/null
python scripts/ncu_summary.py $out/full.ncu-rep "${LABEL:-$tag}: ncu --set full, bench.py --config gpe3d_512, stages 1-4 of one step" 132651000 > $out/ncu_summary.txt 2>&1
cp profiles/ncu_traffic.json $out/ncu_traffic.json
rm -f $out/full.ncu-rep
if [ "${SRC:-1}" = "1" ]; then
  timeout 900 ncu --section SourceCounters --section WarpStateStats --clock-control none -k regex:stage3d_tma -s 9 -c 1 \
    -o $out/src python bench.py --config gpe3d_512 --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > $out/ncu_src.log 2>&1
  ncu -i $out/src.ncu-rep --page source --csv --print-source sass > $out/sass.csv 2>/dev/null
  rm -f $out/src.ncu-rep
fi
if [ "${CONFIGS:-0}" = "1" ]; then
  timeout 900 python scripts/bench_configs.py --json $out/configs.json > $out/configs.txt 2>&1; echo "configs rc=$?"
fi
ls -la $out
