import sys
import torch
sys.path.insert(0, ".")
from paper_2507_11978_b200 import backend as B  # noqa: E402
dev = "cuda:0"
torch.manual_seed(0)
for (m, n, k) in [(256, 256, 32), (128, 128, 64), (256, 256, 256)]:
    a = torch.rand(m, k, device=dev) * 2 - 1
    b = torch.rand(k, n, device=dev) * 2 - 1
    ref = (a.double() @ b.double())
    for at in (False, True):
        for bt in (False, True):
            ta = a.t().contiguous().t() if at else a
            tb = b.t().contiguous().t() if bt else b
            c = torch.zeros(m, n, device=dev)
            B.mm_launch(ta, tb, c, 128, 128, 64)
            torch.cuda.synchronize()
            e = (c.double() - ref).abs()
            print(m, n, k, "A_MN" if at else "A_K ", "B_MN" if bt else "B_K ", f"max err {e.max().item():.3e}",
                  "row0 err", f"{e[0].max().item():.2e}", "row200", f"{e[min(200,m-1)].max().item():.2e}",
                  "col200", f"{e[:, min(200,n-1)].max().item():.2e}")
