import sys
import torch
sys.path.insert(0, ".")
from paper_2507_11978_b200 import backend as B  # noqa: E402
dev = "cuda:0"
M = N = 256
K = 32
A = torch.zeros(M, K, device=dev)
A[torch.arange(M), torch.arange(M) % K] = 1.0          # one-hot: C[m, n] = B[m % 32, n]
kk = torch.arange(K, device=dev).float()[:, None]
nn = torch.arange(N, device=dev).float()[None, :]
for name, Bv in [("code=k", kk.expand(K, N).contiguous()), ("code=n", nn.expand(K, N).contiguous())]:
    for bt in (False, True):
        tb = Bv.t().contiguous().t() if bt else Bv
        c = torch.zeros(M, N, device=dev)
        B.mm_launch(A, tb, c, 128, 128, 64)
        torch.cuda.synchronize()
        ref = A @ Bv
        bad = (c != ref)
        print(name, "B_K " if bt else "B_MN", "bad", int(bad.sum()))
        if bad.any():
            for m in (0, 1, 7, 8, 9, 31, 32, 127, 128, 200):
                print("  row", m, "got", c[m, :12].tolist(), "ref", ref[m, :12].tolist())
