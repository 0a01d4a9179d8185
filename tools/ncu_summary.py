"""Summarise an ncu report: key raw metrics, stall reasons, top stalled SASS lines."""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units, vals = rows[0], rows[1], rows[2]
keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "dram__throughput.avg.pct",
        "launch__registers_per_thread", "sm__warps_active.avg.pct", "smsp__inst_executed.sum",
        "sm__inst_executed_pipe_fp64", "smsp__issue_active.avg.pct", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "lts__t_sectors_srcunit_tex_op_read.sum", "lts__t_sector_hit_rate.pct"]
for i, h in enumerate(hdr):
    if any(h.startswith(k) for k in keys) and "per_second" not in h:
        print(f"{h:80s} {units[i]:10s} {vals[i]}")
print("--- stall reasons (cycles per issued instruction)")
st = [(h, vals[i]) for i, h in enumerate(hdr) if h.startswith("smsp__average_warps_issue_stalled") and h.endswith("per_issue_active.ratio")]
for h, v in sorted(st, key=lambda x: -float(x[1] or 0))[:12]:
    print(f"  {h.replace('smsp__average_warps_issue_stalled_', '').replace('_per_issue_active.ratio', ''):30s} {v}")
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
srows = list(csv.reader(io.StringIO(src)))
h = srows[1]
iS = h.index("Warp Stall Sampling (All Samples)")
data = [r for r in srows[2:] if len(r) > iS and r[iS].isdigit()]
tot = sum(int(r[iS]) for r in data)
print(f"--- top stalled instructions ({tot} samples, {len(data)} SASS lines)")
for r in sorted(data, key=lambda r: -int(r[iS]))[:top]:
    print(f"  {int(r[iS]):6d} {100*int(r[iS])/tot:5.1f}%  {r[0][-5:]}  {r[1][:100]}")
