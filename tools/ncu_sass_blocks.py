"""Executed warp instructions of one kernel's SASS, per basic block (split at
branch targets / after branches): count x block length, in program order."""
import csv, io, re, subprocess, sys
rep, kern = sys.argv[1], sys.argv[2]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass", "-k", f"regex:{kern}"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr, data, seen = None, [], 0
for r in rows:
    if r and r[0] == "Address":
        seen += 1
        hdr = r
        if seen > 1:
            break
        continue
    if hdr and len(r) == len(hdr):
        data.append(r)
ie = hdr.index("Instructions Executed")
tot = sum(int(r[ie] or 0) for r in data)
print(f"total {tot:,}")
blk, cur = [], None
for i, r in enumerate(data):
    ex = int(r[ie] or 0)
    if cur is None or ex != cur[1]:
        cur = [i, ex, 0, r[1].strip()]
        blk.append(cur)
    cur[2] += 1
for b in blk:
    w = b[1] * b[2]
    if w > tot * 0.01:
        print(f"{b[0]:5d} n={b[2]:3d} x{b[1]:>12,} = {w/tot*100:5.1f}%  {b[3][:70]}")
