"""Tuning sweep for the row-streaming kernels (one process per NTB_ROW_RING
setting): device time per launch of softmax / rms_norm over fp16 4096x4096
with rotating input sets (> L2), and a same-bytes torch copy as the
size-matched speed-of-light reference."""
import os
import sys

import torch

sys.path.insert(0, ".")
from paper_2507_11978_b200 import backend as B  # noqa: E402

R = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
C = int(sys.argv[2]) if len(sys.argv) > 2 else 4096
dev = "cuda:0"
nsets = 4
xs = [torch.rand((R, C), device=dev).half() for _ in range(nsets)]
ys = [torch.empty((R, C), device=dev, dtype=torch.float16) for _ in range(nsets)]
w = torch.rand(C, device=dev).half()
steps = 20


def timeit(fn):
    for i in range(3):
        fn(i)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for i in range(steps):
            fn(i)
    g.replay()
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(5):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        g.replay()
        b.record()
        torch.cuda.synchronize()
        best = min(best, a.elapsed_time(b) / steps)
    return best * 1e3


res = {"ring": os.environ.get("NTB_ROW_RING", "auto"),
       "softmax_us": timeit(lambda i: B.softmax_launch(xs[i % nsets], ys[i % nsets], C)),
       "rms_us": timeit(lambda i: B.rms_norm_launch(xs[i % nsets], w, ys[i % nsets], C))}
if os.environ.get("NTB_ROW_RING") is None:
    res["copy_us"] = timeit(lambda i: ys[i % nsets].copy_(xs[i % nsets]))
byt = 2 * R * C * 2
print({k: (round(v, 2) if isinstance(v, float) else v) for k, v in res.items()},
      {k: round(byt / (v * 1e-6) / 1e9) for k, v in res.items() if k.endswith("_us")})
