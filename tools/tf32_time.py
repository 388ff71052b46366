"""Time fp32 mm 4096^3 / bmm 64x1024^3 through the backend (3xTF32 tcgen05)
against torch.mm fp32 (cuBLAS, allow_tf32 False and True).  CUDA events,
CUDA graph of 10 launches, median of 5."""
import statistics
import sys

import torch

sys.path.insert(0, ".")
from paper_2507_11978_b200 import backend as B  # noqa: E402


def t_graph(fn, reps=10):
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        for _ in range(3):
            fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        for _ in range(reps):
            fn()
    ts = []
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        g.replay()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) / reps)
    return statistics.median(ts)


dev = "cuda:0"
M = N = K = 4096
a = torch.rand(M, K, device=dev) * 2 - 1
b = torch.rand(K, N, device=dev) * 2 - 1
c = torch.empty(M, N, device=dev)
fl = 2 * M * N * K
ms = t_graph(lambda: B.mm_launch(a, b, c, 128, 128, 64))
print(f"mm f32 3xTF32 {ms*1e3:.1f} us  {fl/ms/1e9:.1f} TFLOP/s (useful)")
ref = (a.double() @ b.double()).float()
print("max err vs f64", (c - ref).abs().max().item())
torch.backends.cuda.matmul.allow_tf32 = False
ms = t_graph(lambda: torch.mm(a, b, out=c))
print(f"torch.mm fp32 (no tf32) {ms*1e3:.1f} us  {fl/ms/1e9:.1f} TFLOP/s, err {(c-ref).abs().max().item():.2e}")
torch.backends.cuda.matmul.allow_tf32 = True
ms = t_graph(lambda: torch.mm(a, b, out=c))
print(f"torch.mm tf32 {ms*1e3:.1f} us  {fl/ms/1e9:.1f} TFLOP/s, err {(c-ref).abs().max().item():.2e}")
ab = torch.rand(64, 1024, 1024, device=dev) * 2 - 1
bb = torch.rand(64, 1024, 1024, device=dev) * 2 - 1
cb = torch.empty(64, 1024, 1024, device=dev)
ms = t_graph(lambda: B.bmm_launch(ab, bb, cb, 128, 128, 64))
print(f"bmm f32 3xTF32 {ms*1e3:.1f} us  {fl/ms/1e9:.1f} TFLOP/s")
print(B.path_counts())
