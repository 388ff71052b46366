"""Top SASS instructions by warp-stall samples from an .ncu-rep source page."""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
cmd = ["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"]
if len(sys.argv) > 3:
    cmd += ["--kernel-name", f"regex:{sys.argv[3]}"]
out = subprocess.run(cmd, capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]
ia, isrc, iss = hdr.index("Address"), hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)")
body = [r for r in rows[2:] if len(r) == len(hdr) and r[iss].isdigit()]
tot = sum(int(r[iss] or 0) for r in body)
print("total samples", tot)
for i, r in sorted(enumerate(body), key=lambda x: -int(x[1][iss] or 0))[:n]:
    print(f"{i:5d} {int(r[iss]):7d} {100*int(r[iss])/tot:5.1f}%  {r[isrc].strip()[:90]}")
