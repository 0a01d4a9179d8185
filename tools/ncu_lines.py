"""Per-CUDA-source-line warp-stall samples of an ncu report (cuda,sass source view).

usage: python tools/ncu_lines.py report.ncu-rep [top]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
fname, agg, tot = None, [], 0
cur = None
for r in csv.reader(io.StringIO(out)):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] in ("Function Name", "Line No"):
        continue
    if r[0]:  # a source line row (aggregated over its SASS)
        try:
            n = int(r[4])
        except (ValueError, IndexError):
            continue
        tot += n
        if n:
            agg.append((n, f"{fname}:{r[0]}", r[1].strip()[:100]))
print(f"{tot} stall samples")
for n, loc, src in sorted(agg, key=lambda x: -x[0])[:top]:
    print(f"{n:6d} {100 * n / max(tot, 1):5.1f}%  {loc:28s} {src}")
