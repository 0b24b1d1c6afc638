"""Top source lines (CUDA view) by warp-stall samples for one kernel of an ncu report.
    python tools/src_hotspots.py report.ncu-rep kernel_regex [n]"""
import csv
import io
import subprocess
import sys

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source", "cuda",
                      "-k", f"regex:{sys.argv[2]}"], capture_output=True, text=True).stdout
lines = out.splitlines()
# find the header row(s): the report may hold several files
rows = []
cur_file = None
i = 0
while i < len(lines):
    if lines[i].startswith('"File Name"'):
        cur_file = lines[i].split(",", 1)[1].strip('"')
        hdr = next(csv.reader([lines[i + 1]]))
        i += 2
        while i < len(lines) and not lines[i].startswith('"File Name"'):
            r = next(csv.reader([lines[i]]))
            if len(r) == len(hdr):
                rows.append((cur_file, dict(zip(hdr, r))))
            i += 1
    else:
        i += 1
key = "Warp Stall Sampling (All Samples)"
tot = sum(float(r.get(key) or 0) for _, r in rows)
top = sorted(rows, key=lambda fr: -float(fr[1].get(key) or 0))[: int(sys.argv[3]) if len(sys.argv) > 3 else 25]
for f, r in top:
    s = float(r.get(key) or 0)
    print(f"{s / tot:6.1%} {f.split('/')[-1]}:{r['Line No']:>5}  {r['Source'].strip()[:100]}")
