"""Top stalled SASS instructions of one kernel in an ncu report.
    python tools/sass_hot.py report kernel_regex [n]"""
import csv
import io
import subprocess
import sys

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "-k", f"regex:{sys.argv[2]}"],
                     capture_output=True, text=True).stdout
lines = out.splitlines()
rows = list(csv.reader(io.StringIO("\n".join(lines[1:]))))
hdr = rows[0]
si, st, nst = hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Warp Stall Sampling (Not-issued Samples)")
data = []
for i, r in enumerate(rows[1:]):
    try:
        data.append((int(r[st]), int(r[nst]), i, r[si].strip()))
    except (ValueError, IndexError):
        pass
tot = sum(d[0] for d in data)
for s, ns, i, src in sorted(data, reverse=True)[: int(sys.argv[3]) if len(sys.argv) > 3 else 30]:
    print(f"{s / tot:6.2%} (not-issued {ns / tot:6.2%}) #{i:5d}  {src[:90]}")
