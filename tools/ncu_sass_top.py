"""Top SASS instructions of one kernel in an .ncu-rep by executed warp
instructions and by stall samples (ncu --page source --print-source sass)."""
import csv, io, subprocess, sys
rep = sys.argv[1]
kern = sys.argv[2] if len(sys.argv) > 2 else None
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
cmd = ["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"]
if kern:
    cmd += ["-k", f"regex:{kern}"]
out = subprocess.run(cmd, capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = None
data = []
for r in rows:
    if r and r[0] == "Address":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        data.append(r)
ie = hdr.index("Instructions Executed")
ss = hdr.index("Warp Stall Sampling (All Samples)")
tot = sum(int(r[ie] or 0) for r in data)
tots = sum(int(r[ss] or 0) for r in data)
print(f"instructions {tot:,}  samples {tots:,}  sass lines {len(data)}")
for i, r in enumerate(data):
    r.append(i)
for r in data:
    ex, sm = int(r[ie] or 0), int(r[ss] or 0)
    if ex > tot * 0.004 or sm > tots * 0.01:
        print(f"{r[-1]:5d} {ex/tot*100:5.1f}% {sm/max(tots,1)*100:5.1f}%  {r[1].strip()[:90]}")
