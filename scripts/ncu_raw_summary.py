#!/usr/bin/env python
"""Compact per-launch summary of an `ncu --page raw --csv` export: duration, DRAM bytes, L2 hit
rate, issue activity, occupancy, pipe utilisation and the top warp-stall reasons.
    python scripts/ncu_raw_summary.py RAW.csv [points_per_launch] > summary.json"""
import csv
import json
import sys

KEYS = {
    "gpu__time_duration.sum": "duration",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "lts__t_sector_hit_rate.pct": "l2_hit_pct",
    "sm__inst_issued.avg.pct_of_peak_sustained_active": "issue_active_pct",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "occupancy_pct",
    "smsp__inst_executed.sum": "warp_inst",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active": "fp64_pipe_pct",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed": "lsu_shared_wavefronts_pct",
    "sm__cycles_active.avg": "sm_cycles_active",
    "gpc__cycles_elapsed.max": "gpc_cycles_elapsed",
    "launch__registers_per_thread": "registers",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed": "dram_throughput_pct",
}


def main():
    rows = list(csv.reader(open(sys.argv[1])))
    hdr, units = rows[0], rows[1]
    pts = float(sys.argv[2]) if len(sys.argv) > 2 else None
    out = []
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        u = dict(zip(hdr, units))
        e = {"kernel": d.get("Kernel Name", "")[:90]}
        for k, name in KEYS.items():
            if k in d and d[k] not in ("", "n/a"):
                try:
                    v = float(d[k].replace(",", ""))
                except ValueError:
                    continue
                unit = u.get(k, "")
                if unit in ("Kbyte", "Mbyte", "Gbyte"):
                    v *= {"Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}[unit]
                if name == "duration":
                    name = f"duration_{unit}"
                e[name] = round(v, 3)
        st = []
        for k in hdr:
            if "pcsamp_warps_issue_stalled" in k and not k.endswith("not_issued"):
                try:
                    v = float(d[k].replace(",", ""))
                except ValueError:
                    continue
                if v > 0:
                    st.append((v, k.replace("smsp__pcsamp_warps_issue_stalled_", "")))
        tot = sum(v for v, _ in st) or 1
        e["top_stalls_pct"] = {k: round(100 * v / tot, 1) for v, k in sorted(st, reverse=True)[:6]}
        if pts and "dram_read" in e:
            e["dram_B_per_point"] = round((e["dram_read"] + e.get("dram_write", 0)) / pts, 2)
        if "sm_cycles_active" in e and "gpc_cycles_elapsed" in e:
            e["sm_active_frac"] = round(e["sm_cycles_active"] / e["gpc_cycles_elapsed"], 3)
        out.append(e)
    json.dump(out, sys.stdout, indent=1)


if __name__ == "__main__":
    main()
