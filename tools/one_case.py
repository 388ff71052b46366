"""Run one small case of a family on cuda:0 (debug helper for sanitizer runs)."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2507_11978_b200 import backend as B  # noqa: E402

kind = sys.argv[1]
dev = "cuda:0"
rng = np.random.default_rng(0)


def T(shape):
    return torch.from_numpy(rng.uniform(-1, 1, shape).astype(np.float32)).to(dev).half()


if kind == "conv":
    n, c, h, w, k, r, s = (int(x) for x in sys.argv[2:9])
    x, f = T((n, c, h, w)), T((k, c, r, s))
    y = torch.zeros((n, k, h - r + 1, w - s + 1), device=dev, dtype=torch.float16)
    B.conv2d_launch(x, f, y, 128, 128, 64)
    torch.cuda.synchronize()
    ref = torch.nn.functional.conv2d(x.float(), f.float())
    print("conv max err", (y.float() - ref).abs().max().item(), B.path_counts())
elif kind == "sdpa":
    b, h, sq, d = (int(x) for x in sys.argv[2:6])
    q, kk, v = T((b, h, sq, d)), T((b, h, sq, d)), T((b, h, sq, d))
    o = torch.zeros_like(q)
    B.sdpa_launch(q, kk, v, o, 128, 128)
    torch.cuda.synchronize()
    # math reference (cuBLAS GEMMs): PyTorch's own SDPA kernels would be in
    # the sanitizer's report too
    ref = torch.softmax(q.float() @ kk.float().transpose(-1, -2) / d ** 0.5, -1) @ v.float()
    print("sdpa max err", (o.float() - ref).abs().max().item(), B.path_counts())
elif kind == "sdpa_rope":
    b, s_, h, d = (int(x) for x in sys.argv[2:6])
    base = [T((b, s_, h, d)) for _ in range(3)]
    ang = torch.rand((s_, d // 2), device=dev) * 6 - 3
    sn, cs = torch.sin(ang).half(), torch.cos(ang).half()
    q, kk, v = (x.transpose(1, 2) for x in base)
    o = torch.zeros((b, h, s_, d), device=dev, dtype=torch.float16)
    B.sdpa_rope_launch(q, kk, v, sn, cs, sn, cs, o, 128, 128)
    torch.cuda.synchronize()

    def rot(x):
        x = x.float()
        x0, x1 = x[..., :d // 2], x[..., d // 2:]
        c, s = cs.float(), sn.float()
        return torch.cat([x0 * c - x1 * s, x0 * s + x1 * c], -1).half().float()

    ref = torch.softmax(rot(q) @ rot(kk).transpose(-1, -2) / d ** 0.5, -1) @ v.float()
    print("sdpa_rope max err", (o.float() - ref).abs().max().item(), B.path_counts())
elif kind == "mm":
    m, n, k = (int(x) for x in sys.argv[2:5])
    a, b = T((m, k)), T((k, n))
    c = torch.zeros((m, n), device=dev, dtype=torch.float16)
    B.mm_launch(a, b, c, 128, 128, 64)
    torch.cuda.synchronize()
    print("mm", m, n, k, "max err", (c.float() - a.float() @ b.float()).abs().max().item(),
          {k_: v for k_, v in B.path_counts().items() if v})
elif kind == "mm32":   # fp32 operands: the 3xTF32 tcgen05 kernel
    m, n, k = (int(x) for x in sys.argv[2:5])
    a = torch.rand((m, k), device=dev) * 2 - 1
    b = torch.rand((k, n), device=dev) * 2 - 1
    c = torch.zeros((m, n), device=dev)
    B.mm_launch(a, b, c, 128, 128, 64)
    torch.cuda.synchronize()
    ref = (a.double() @ b.double()).float()
    print("mm32", m, n, k, "max err", (c - ref).abs().max().item(),
          {k_: v for k_, v in B.path_counts().items() if v})
elif kind == "bmm":
    bt, m, n, k = (int(x) for x in sys.argv[2:6])
    a, b = T((bt, m, k)), T((bt, k, n))
    c = torch.zeros((bt, m, n), device=dev, dtype=torch.float16)
    for _ in range(3):
        B.bmm_launch(a, b, c, 128, 128, 64)
    torch.cuda.synchronize()
    print("bmm max err", (c[:2].float() - a[:2].float() @ b[:2].float()).abs().max().item())
elif kind == "rows":
    r, c = (int(x) for x in sys.argv[2:4])
    x = T((r, c))
    w = T((c,))
    y = torch.zeros_like(x)
    B.softmax_launch(x, y, c)
    torch.cuda.synchronize()
    print("softmax max err", (y.float() - torch.softmax(x.float(), -1)).abs().max().item())
    B.rms_norm_launch(x, w, y, c)
    torch.cuda.synchronize()
    ref = x.float() * torch.rsqrt(x.float().pow(2).mean(-1, keepdim=True) + 1e-6) * w.float()
    print("rms max err", (y.float() - ref).abs().max().item())
elif kind == "ew":
    n = int(sys.argv[2])
    a, b = T((n,)).float(), T((n,)).float()
    o = torch.zeros_like(a)
    B.add_launch(a, b, o, 1024)
    torch.cuda.synchronize()
    print("add max err", (o - (a + b)).abs().max().item())
elif kind == "rope":
    bb, s, h, d = (int(x) for x in sys.argv[2:6])
    x = T((bb, s, h, d))
    ang = torch.rand((s, d // 2), device=dev) * 6 - 3
    sn, cs = torch.sin(ang).half(), torch.cos(ang).half()
    o = torch.zeros_like(x)
    B.rope_launch(x, sn, cs, o, d // 2)
    torch.cuda.synchronize()
    x0, x1 = x.float()[..., : d // 2], x.float()[..., d // 2:]
    c2, s2 = cs.float()[None, :, None, :], sn.float()[None, :, None, :]
    ref = torch.cat([x0 * c2 - x1 * s2, x0 * s2 + x1 * c2], -1)
    print("rope max err", (o.float() - ref).abs().max().item())
