"""Summarise an `ncu --set full` capture of the stage kernels into profiles/.

    python scripts/ncu_summary.py gpurun_out/<tag>/prof.ncu-rep <capture-label> <interior-points-per-launch>

Writes profiles/ncu_traffic.json[<variant>] = dram bytes (read + write) per interior point
per stage launch, averaged over the captured launches (one RK4 step = stages 1-4), which
bench.py scales to its own launch size for the roofline "traffic" field, and prints a
per-launch table.
"""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def main():
    rep, label, pts = sys.argv[1], sys.argv[2], float(sys.argv[3])
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    ix = {h: i for i, h in enumerate(hdr)}

    def val(r, k):
        v = r[ix[k]].replace(",", "")
        u = units[ix[k]]
        x = float(v)
        scale = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0, "Tbyte": 1e12}.get(u, 1.0)
        if k.startswith("gpu__time"):
            scale = {"ms": 1e-3, "us": 1e-6, "ns": 1e-9, "s": 1.0}.get(u, 1.0)
        return x * scale
    out = []
    for r in rows[2:]:
        name = r[ix["Kernel Name"]]
        rd, wr = val(r, "dram__bytes_read.sum"), val(r, "dram__bytes_write.sum")
        t = val(r, "gpu__time_duration.sum")
        out.append((name, rd, wr, t))
        print(f"{name[:60]:60s} read {rd/pts:6.1f} B/pt  write {wr/pts:6.1f} B/pt  {t*1e3:8.3f} ms  "
              f"{(rd+wr)/t/1e9:7.1f} GB/s")
    variant = "stage3d_tma" if "stage3d_tma" in out[0][0] else ("stage3d_stream" if "stream" in out[0][0] else "other")
    per_pt = sum(o[1] + o[2] for o in out) / len(out) / pts
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    d = json.load(open(path)) if os.path.exists(path) else {}
    d[variant] = {"dram_bytes_per_point_stage": round(per_pt, 2), "capture": label, "launches": len(out)}
    json.dump(d, open(path, "w"), indent=1)
    print(f"{variant}: {per_pt:.2f} dram B per interior point per stage launch (avg of {len(out)})")


if __name__ == "__main__":
    main()
