"""SASS lines of an .ncu-rep with excess shared-memory wavefronts (bank
conflicts), with the CUDA source line they map to.

    python tools/ncu_conflicts.py gpurun_out/x.ncu-rep [N] [kernel-regex]
"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 20
base = ["ncu", "-i", rep, "--page", "source", "--csv"]
if len(sys.argv) > 3:
    base += ["--kernel-name", f"regex:{sys.argv[3]}"]


def table(kind):
    out = subprocess.run(base + ["--print-source", kind], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    i = next(k for k, r in enumerate(rows) if r and r[0] in ("Address", "# Address", "Line"))
    return rows[i], [r for r in rows[i + 1:] if len(r) == len(rows[i])]


hdr, body = table("sass")
ix = {h: i for i, h in enumerate(hdr)}
exc = ix["L1 Wavefronts Shared Excessive"]
tot = sum(float(r[exc] or 0) for r in body)
print(f"excess shared wavefronts: {tot:.0f}")
for r in sorted(body, key=lambda r: -float(r[exc] or 0))[:n]:
    if float(r[exc] or 0) == 0:
        break
    print(f"{float(r[exc]):10.0f}  ideal {r[ix['L1 Wavefronts Shared Ideal']]:>9}  {r[ix['Address']]}  {r[ix['Source']].strip()[:80]}")
try:
    hdr, body = table("cuda")
    ix = {h: i for i, h in enumerate(hdr)}
    exc = ix["L1 Wavefronts Shared Excessive"]
    print("-- by CUDA source line")
    for r in sorted(body, key=lambda r: -float(r[exc] or 0))[:n]:
        if float(r[exc] or 0) == 0:
            break
        print(f"{float(r[exc]):10.0f}  {r[ix.get('Line', 0)]}  {r[ix['Source']].strip()[:90]}")
except Exception as e:  # noqa: BLE001
    print("cuda view unavailable:", e)
