#!/bin/bash
# tile order A/B at 1024^3: bench + DRAM bytes of the 4 stage launches per NLSE_TILE_BAND value
out=gpurun_out/${TAG:-band}; mkdir -p $out
python -c "import __graft_entry__ as g; g.build()" > $out/build.log 2>&1 || { echo BUILD FAILED; exit 1; }
for b in ${BANDS:-0 2 4 8}; do
  NLSE_TILE_BAND=$b timeout 600 python bench.py --steps 20 --no-e2e --no-cpu-baseline > $out/bench_$b.json 2>> $out/bench.err
  python scripts/brief.py "band=$b" < $out/bench_$b.json
done
for b in ${BANDS:-0 2 4 8}; do
  NLSE_TILE_BAND=$b timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
    -k regex:stage3d_tma -s 64 -c 4 --csv --log-file $out/dram_$b.csv \
    python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > $out/ncu_$b.log 2>&1
  python - $out/dram_$b.csv $b <<'PY'
import csv,sys
rows=[r for r in csv.reader(open(sys.argv[1])) if len(r)>10]
h=rows[0]; i_m=h.index("Metric Name"); i_v=h.index("Metric Value")
rd=sum(float(r[i_v].replace(',','')) for r in rows[1:] if r[i_m]=="dram__bytes_read.sum")
wr=sum(float(r[i_v].replace(',','')) for r in rows[1:] if r[i_m]=="dram__bytes_write.sum")
u=[r[h.index("Metric Unit")] for r in rows[1:] if r[i_m]=="dram__bytes_read.sum"][0]
scale={"byte":1,"Kbyte":1e3,"Mbyte":1e6,"Gbyte":1e9}.get(u,1)
n=1022*1022*1022
print(f"band={sys.argv[2]} DRAM bytes per interior point per stage (avg of 4 launches): {(rd+wr)*scale/4/n:.2f}  (read {rd*scale/4/n:.2f}, write {wr*scale/4/n:.2f})")
PY
done
