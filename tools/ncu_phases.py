"""Instruction / stall shares of one kernel by code region: regions start at
source lines containing the given marker substrings (the report's own
imported source), helpers outside the kernel body are listed per line.
    python tools/ncu_phases.py rep.ncu-rep <kernel-regex> <first-line-marker> <marker>...
"""
import collections
import csv
import io
import subprocess
import sys

rep, kern, *marks = sys.argv[1:]
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", "regex:" + kern,
                      "--print-source", "cuda,sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
src = {}
data = []
for r in rows:
    if len(r) > 8 and r[0].isdigit():
        src[int(r[0])] = r[1]
        if r[2] == "-":
            data.append((int(r[0]), int(r[7] or 0), int(r[4] or 0)))
pos = []
for m in marks:
    ln = next((k for k in sorted(src) if m in src[k]), None)
    pos.append((m, ln))
pos = [p for p in pos if p[1] is not None]
pos.sort(key=lambda p: p[1])
end = max(src)
agg, st = collections.Counter(), collections.Counter()
for ln, i, s in data:
    name = None
    for k, (m, p) in enumerate(pos):
        q = pos[k + 1][1] if k + 1 < len(pos) else None
        if ln >= p and (q is None or ln < q):
            name = m[:40]
    if name is None or ln < pos[0][1]:
        name = f"helper L{ln}: {src[ln].strip()[:60]}"
    agg[name] += i
    st[name] += s
ti, ts = sum(agg.values()) or 1, sum(st.values()) or 1
print(f"warp-instructions {ti}")
for k, v in agg.most_common(40):
    print(f"{100 * v / ti:5.1f}% inst {100 * st[k] / ts:5.1f}% stall  {k}")
