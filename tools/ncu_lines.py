"""Per-source-line stall samples and instruction counts of one kernel from an
ncu report (needs -lineinfo):  python tools/ncu_lines.py rep.ncu-rep <kernel-regex> [top]"""
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", "regex:" + kern,
                      "--print-source", "cuda,sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
data = []
fname = "?"
for r in rows:
    if len(r) >= 2 and r[0] == "File Path":  # the page lists each source file in turn
        fname = r[1].rsplit("/", 1)[-1]
        continue
    if len(r) > 8 and r[0].isdigit() and r[2] == "-":
        try:
            data.append((int(r[4] or 0), int(r[7] or 0), f"{fname}:{r[0]}", r[1][:100]))
        except ValueError:
            pass
ts = sum(x[0] for x in data) or 1
ti = sum(x[1] for x in data) or 1
print(f"samples {ts}  warp-instructions {ti}")
for s, i, ln, src in sorted(data, reverse=True)[:top]:
    print(f"{100 * s / ts:5.1f}% stall  {100 * i / ti:5.1f}% inst  {ln:<20} {src}")
