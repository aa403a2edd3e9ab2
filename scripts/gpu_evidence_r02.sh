#!/bin/bash
# Round-2 evidence pass: -m gpu suite, smoke, the default bench line, the ncu launch list of the
# same command, one `ncu --set full` capture of the four stage launches of one step at 512^3
# (summarised into profiles/ncu_traffic.json by scripts/ncu_summary.py), DRAM bytes of the four
# stage launches at 1024^3 (the bench size), and all BASELINE configurations.
tag=${TAG:-r02ev}; out=gpurun_out/$tag; mkdir -p $out
python -c "import __graft_entry__ as g; g.build()" > $out/build.log 2>&1 || { echo BUILD FAILED; exit 1; }
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,power.limit --format=csv > $out/nvsmi.txt 2>&1
if [ "${TESTS:-1}" = "1" ]; then
  timeout 1800 python -m pytest tests -m gpu -q --timeout 600 > $out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 $out/pytest_gpu.log
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $out/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 $out/smoke.log
fi
timeout 900 python bench.py > $out/bench.json 2> $out/bench.err; echo "bench rc=$?"; python scripts/brief.py default < $out/bench.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $out/launches.csv \
  python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > $out/ncu_launch.log 2>&1; echo "ncu launches rc=$?"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:stage3d_tma -s 8 -c 4 \
  -o $out/full python bench.py --config gpe3d_512 --steps 2 --warmup 1 --no-e2e --no-cpu-baseline \
  > $out/ncu_full.log 2>&1; echo "ncu full rc=$?"
ncu -i $out/full.ncu-rep --page raw --csv > $out/full_raw.csv 2>/dev/null
python scripts/ncu_summary.py $out/full.ncu-rep "${LABEL:-$tag}: ncu --set full, bench.py --config gpe3d_512, stages 1-4 of one step" 132651000 > $out/ncu_summary.txt 2>&1
cp profiles/ncu_traffic.json $out/ncu_traffic.json
rm -f $out/full.ncu-rep
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
  -k regex:stage3d_tma -s 64 -c 4 --csv --log-file $out/dram_1024.csv \
  python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > $out/ncu_dram_1024.log 2>&1; echo "ncu dram 1024 rc=$?"
if [ "${CONFIGS:-1}" = "1" ]; then
  timeout 900 python scripts/bench_configs.py --json $out/configs.json > $out/configs.txt 2>&1; echo "configs rc=$?"; tail -12 $out/configs.txt
fi
ls -la $out
