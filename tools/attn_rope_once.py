"""One sdpa_rope launch at the bench shape (B32 H32 S4096 D128), timed; for
debug builds (NTB_LIB_VARIANT) that print per-launch statistics."""
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_2507_11978_b200 import backend as B  # noqa: E402

dev = "cuda:0"
b = int(sys.argv[1]) if len(sys.argv) > 1 else 32
shp = (b, 4096, 32, 128)
q, k, v = (torch.rand(shp, device=dev).half() for _ in range(3))
ang = torch.rand((4096, 64), device=dev) * 6 - 3
sn, cs = torch.sin(ang).half(), torch.cos(ang).half()
o = torch.empty((b, 32, 4096, 128), device=dev, dtype=torch.float16)
T = lambda x: x.transpose(1, 2)  # noqa: E731
for i in range(3):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    B.sdpa_rope_launch(T(q), T(k), T(v), sn, cs, sn, cs, o, 128, 128)
    e1.record()
    torch.cuda.synchronize()
    print(f"sdpa_rope {e0.elapsed_time(e1):.3f} ms", flush=True)
