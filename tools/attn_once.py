"""One sdpa launch at B H S D (default the bench shape), timed with events;
for debug builds (NTB_LIB_VARIANT) that print per-launch traces."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2507_11978_b200 import backend as B  # noqa: E402

b, h, s, d = (int(x) for x in (sys.argv[1:5] if len(sys.argv) >= 5 else (32, 32, 4096, 128)))
q, k, v = (torch.rand((b, h, s, d), device="cuda").half() for _ in range(3))
o = torch.empty_like(q)
for i in range(3):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    B.sdpa_launch(q, k, v, o, 128, 128)
    e1.record()
    torch.cuda.synchronize()
    print(f"sdpa {e0.elapsed_time(e1):.3f} ms", flush=True)
