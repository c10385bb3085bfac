"""Summary of one kernel's `ncu --set full` capture as JSON (the figures the bench's roofline
line and DESIGN.md quote):  python tools/ncu_summary.py gpurun_out/prof_x.ncu-rep > profiles/x.json"""
import csv, json, subprocess, sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active",
        "lts__t_sector_hit_rate.pct", "launch__registers_per_thread", "launch__grid_size", "launch__block_size"]
raw = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
h, u, v = rows[0], rows[1], rows[2]
out = {"capture": sys.argv[1].split("/")[-1], "kernel": v[h.index("Kernel Name")] if "Kernel Name" in h else None}
for k in KEYS:
    if k in h:
        out[k] = {"unit": u[h.index(k)], "value": v[h.index(k)]}
print(json.dumps(out, indent=1))
