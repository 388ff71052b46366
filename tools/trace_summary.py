"""Average the per-phase clock64 stamps printed by an NTB_ATTN_TRACE build
(tools/one_case.py sdpa ...) over the steady-state tiles."""
import re
import sys

rows = [ln for ln in open(sys.argv[1]) if ln.startswith("j=")]
vals = []
for ln in rows[4:30]:
    nums = [int(x) for x in re.findall(r"[-+]?\d+", ln.split("|", 1)[1])]
    vals.append(nums)
if not vals:
    sys.exit("no trace rows")
n = len(vals)
avg = [sum(v[i] for v in vals) / n for i in range(len(vals[0]))]
cyc = (int(re.findall(r"wait@\s*(-?\d+)", rows[29])[0]) - int(re.findall(r"wait@\s*(-?\d+)", rows[4])[0])) / 25
print(f"cycle/j {cyc:.0f} | g0 wait {avg[2]:.0f} ld {avg[3]:.0f} max {avg[4]:.0f} h0 {avg[5]:.0f} "
      f"h1 {avg[6]:.0f} | g1 wait {avg[8]:.0f} max {avg[10]:.0f} h0 {avg[11]:.0f} h1 {avg[12]:.0f}")
