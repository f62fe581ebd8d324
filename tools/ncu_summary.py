"""Turn an `ncu --set full` capture of the top kernels into the summary
bench.py reads (profiles/ncu_traffic.json): per kernel, DRAM bytes per
launch (dram__bytes_read.sum + dram__bytes_write.sum), issue-slot and
warp-occupancy percentages, instructions and duration.

    ncu -i gpurun_out/full.ncu-rep --page raw --csv > profiles/rNN_ncu_full_top_kernels.csv
    python tools/ncu_summary.py profiles/rNN_ncu_full_top_kernels.csv > profiles/ncu_traffic.json
"""
import csv
import json
import sys

KEYS = {"bin_front": "bin_front_kernel", "blend_forward": "blend_forward_",
        "ssim_bwd": "ssim_bwd_kernel", "backward": "backward_quad_kernel",
        "chain_adam": "chain_adam_kernel", "ssim_fwd": "ssim_fwd_kernel",
        "preprocess": "preprocess_kernel"}
SCALE = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-3,
         "usecond": 1.0, "msecond": 1e3}

path = sys.argv[1]
rows = list(csv.reader(open(path)))
h, units = rows[0], rows[1]


def val(row, name):
    i = h.index(name)
    return float(row[i].replace(",", "")) * SCALE.get(units[i], 1.0)


out = {}
for r in rows[2:]:
    name = r[h.index("Kernel Name")]
    for key, pat in KEYS.items():
        if pat in name and key not in out:
            out[key] = {
                "dram_bytes": int(val(r, "dram__bytes_read.sum") + val(r, "dram__bytes_write.sum")),
                "issue_slots_pct": round(val(r, "sm__inst_issued.avg.pct_of_peak_sustained_active"), 2),
                "warps_active_pct": round(val(r, "sm__warps_active.avg.pct_of_peak_sustained_active"), 2),
                "inst_executed": int(val(r, "smsp__inst_executed.sum")),
                "duration_us": round(val(r, "gpu__time_duration.sum"), 2),
            }
out["_source"] = (f"{path}: ncu --set full --clock-control none on tools/profile_step.py (one "
                  "launch each); dram_bytes = dram__bytes_read.sum + dram__bytes_write.sum, "
                  "issue_slots_pct = sm__inst_issued.avg.pct_of_peak_sustained_active, "
                  "warps_active_pct = sm__warps_active.avg.pct_of_peak_sustained_active")
print(json.dumps(out, indent=1))
