#!/bin/bash
# Round-2 final evidence pass (after the 2D warp-strip kernel): -m gpu suite + smoke, the default
# bench line, its ncu launch list, DRAM bytes of the four stage launches at 1024^3, ncu --set full
# of the 2D strip kernel (trap2d) and of the 3D stage kernel (512^3), all BASELINE configurations,
# the size sweeps.  (compute-sanitizer is closed on this pool.)
tag=${TAG:-r02fin}; out=gpurun_out/$tag; mkdir -p $out
python -c "import __graft_entry__ as g; g.build()" > $out/build.log 2>&1 || { echo BUILD FAILED; exit 1; }
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,power.limit --format=csv > $out/nvsmi.txt 2>&1
if [ "${TESTS:-1}" = "1" ]; then
  timeout 1800 python -m pytest tests -m gpu -q --timeout 600 > $out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 $out/pytest_gpu.log
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $out/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 $out/smoke.log
fi
timeout 900 python bench.py > $out/bench.json 2> $out/bench.err; echo "bench rc=$?"; python scripts/brief.py default < $out/bench.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $out/launches.csv \
  python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > $out/ncu_launch.log 2>&1; echo "ncu launches rc=$?"
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
  -k regex:stage3d_tma -s 64 -c 4 --csv --log-file $out/dram_1024.csv \
  python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > $out/ncu_dram_1024.log 2>&1; echo "ncu dram 1024 rc=$?"
timeout 900 ncu --set full --clock-control none --cache-control none --import-source on -k regex:stage2d_strip -s 40 -c 4 \
  -o $out/full2d python bench.py --config trap2d --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > $out/ncu_full2d.log 2>&1; echo "ncu full 2d rc=$?"
ncu -i $out/full2d.ncu-rep --page raw --csv > $out/full2d_raw.csv 2>/dev/null
ncu -i $out/full2d.ncu-rep --page details > $out/full2d_details.txt 2>/dev/null
rm -f $out/full2d.ncu-rep
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:stage3d_tma -s 8 -c 4 \
  -o $out/full3d python bench.py --config gpe3d_512 --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > $out/ncu_full3d.log 2>&1; echo "ncu full 3d rc=$?"
ncu -i $out/full3d.ncu-rep --page raw --csv > $out/full3d_raw.csv 2>/dev/null
ncu -i $out/full3d.ncu-rep --page details > $out/full3d_details.txt 2>/dev/null
rm -f $out/full3d.ncu-rep
if [ "${CONFIGS:-1}" = "1" ]; then
  timeout 900 python scripts/bench_configs.py --json $out/configs.json > $out/configs.txt 2>&1; echo "configs rc=$?"; tail -12 $out/configs.txt
  timeout 1200 python scripts/bench_sizes.py --set all > $out/sizes.jsonl 2> $out/sizes.err; echo "sizes rc=$?"; tail -12 $out/sizes.jsonl
fi
ls -la $out
