"""Run one kernel family back-to-back for ~N seconds (for clock / power sampling)."""
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_2507_11978_b200 import backend as B  # noqa: E402

kind, secs = sys.argv[1], float(sys.argv[2])
dev = "cuda:0"
if kind == "sdpa":
    shp = (32, 32, 4096, 128)
    q, k, v = (torch.randn(shp, device=dev, dtype=torch.float16) for _ in range(3))
    o = torch.empty_like(q)
    fn = lambda: B.sdpa_launch(q, k, v, o, 128, 128)  # noqa: E731
    flops = 4 * 32 * 32 * 4096 * 4096 * 128
elif kind == "mm":
    a, b = (torch.randn(4096, 4096, device=dev, dtype=torch.float16) for _ in range(2))
    c = torch.empty_like(a)
    fn = lambda: B.mm_launch(a, b, c, 128, 128, 64)  # noqa: E731
    flops = 2 * 4096 ** 3
fn()
torch.cuda.synchronize()
t0 = time.time()
n = 0
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
while time.time() - t0 < secs:
    for _ in range(5):
        fn()
    n += 5
    torch.cuda.synchronize()
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / n
print(f"{kind}: {n} calls, {ms:.3f} ms/call, {flops / ms / 1e9:.1f} TFLOP/s")
