"""profiles/traffic.json from the ncu CSV of tools/traffic_probe.py: per bench
key, the DRAM bytes of its launches, reads from dram__bytes_read and writes
as max(dram__bytes_write, 32 B x lts__t_sectors_srcunit_tex_op_write) - writes still
dirty in the 126 MB L2 when a kernel ends never reach DRAM inside the
capture, so the L2 write sectors stand in for them.

    python tools/make_traffic.py gpurun_out/r2_traffic.csv "softmax,rms_norm,..."
"""
import csv
import io
import json
import sys
from collections import defaultdict

L2_BYTES = 126 * 1024 * 1024
rows = [r for r in csv.reader(io.StringIO(open(sys.argv[1]).read())) if r]
hdr = next(r for r in rows if "ID" in r and "Metric Name" in r)
ix = {h: i for i, h in enumerate(hdr)}
data = defaultdict(dict)
names = {}
for r in rows[rows.index(hdr) + 1:]:
    if len(r) != len(hdr):
        continue
    lid = int(r[ix["ID"]])
    names[lid] = r[ix["Kernel Name"]]
    val = float(r[ix["Metric Value"]].replace(",", ""))
    unit = r[ix["Metric Unit"]]
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "sector": 1, "nsecond": 1,
             "usecond": 1e3, "msecond": 1e6}.get(unit, 1)
    data[lid][r[ix["Metric Name"]]] = val * scale
order = sys.argv[2].split(",")
# the launches of each key are those between consecutive synchronisations;
# kernels are attributed by name: every key's main kernel families
FAMILY = {"softmax": "row_stream", "rms_norm": "row_stream", "add_2^20": "ew_vec",
          "add_2^24": "ew_stream", "silu_2^24": "ew_stream", "mm": "gemm_pair", "addmm": "gemm_pair",
          "bmm": "gemm_pair", "mm_f32": "gemm_tf32", "bmm_f32": "gemm_tf32",
          "conv2d": "conv_fused", "conv2d_f32": "gemm_tf32", "sdpa": "attn_fwd", "rope": "rope_vec",
          "sdpa_rope": "attn_fwd"}
def traffic(d):
    # bytes written = between the DRAM write counter and that plus one L2 of
    # dirty lines still resident at kernel end; the SM-sourced L2 write
    # sectors (32 B each) estimate it, capped by that bound (partial-sector
    # stores count a sector per store)
    dw = d.get("dram__bytes_write.sum", 0)
    wr = max(dw, min(32 * d.get("lts__t_sectors_srcunit_tex_op_write.sum", 0), dw + L2_BYTES))
    return d.get("dram__bytes_read.sum", 0) + wr


ids = sorted(data)
out, seen = {}, defaultdict(int)
k = 0
for key in order:
    fam = FAMILY[key]
    while k < len(ids) and fam not in names[ids[k]]:
        k += 1
    if k == len(ids):
        break
    # sdpa_rope runs one attention launch per batch chunk (each after its
    # rope_vec K pre-pass): the key's traffic is the sum of those launches
    group = [ids[k]]
    if key == "sdpa_rope":
        j = k + 1
        while j < len(ids) and ("attn_fwd" in names[ids[j]] or "rope_vec" in names[ids[j]]):
            if "attn_fwd" in names[ids[j]]:
                group.append(ids[j])
            j += 1
        k = j - 1
    tot = 0
    for lid in group:
        tot += traffic(data[lid])
    out[key] = int(tot)
    k += 1
out["_note"] = ("per launch, ncu on tools/traffic_probe.py (cold L2 per replay): "
                "dram__bytes_read.sum + writes "
                "of the key's main kernel, with writes = max(W, min(32 B x L2 write sectors, W + "
                "126 MB)), W = dram__bytes_write.sum: writes left dirty in the L2 at kernel end "
                "never reach DRAM inside the capture (the L2 write sectors count them), but at "
                "most one L2 of them can (partial-sector stores, e.g. the attention epilogue's "
                "16 B per row, count one sector per store). sdpa_rope: its attention launches "
                "summed, one per batch chunk of the rotated-K workspace (the K pre-pass is a "
                "separate rope_vec launch per chunk).")
json.dump(out, open("profiles/traffic.json", "w"), indent=1)
print(json.dumps(out, indent=1))
