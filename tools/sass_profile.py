"""Aggregate an ncu source page (SASS view) by opcode: executed warp instructions
and stall samples.   python tools/sass_profile.py report.ncu-rep kernel_regex"""
import collections
import csv
import io
import re
import subprocess
import sys

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "-k", f"regex:{sys.argv[2]}"],
                     capture_output=True, text=True).stdout
lines = out.splitlines()
rows = list(csv.reader(io.StringIO("\n".join(lines[1:]))))
hdr = rows[0]
si, ie, st = hdr.index("Source"), hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
cnt, stall = collections.Counter(), collections.Counter()
for r in rows[1:]:
    if len(r) <= max(si, ie, st):
        continue
    src = r[si].strip()
    m = re.match(r"(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)", src)
    if not m:
        continue
    op = m.group(1)
    try:
        cnt[op] += int(r[ie])
        stall[op] += int(r[st])
    except ValueError:
        pass
tot, tst = sum(cnt.values()), sum(stall.values())
print(f"total warp instructions {tot}, stall samples {tst}")
for op, n in cnt.most_common(28):
    print(f"  {op:10s} {n:12d} {n / tot:6.1%}   stalls {stall[op] / max(tst, 1):6.1%}")
