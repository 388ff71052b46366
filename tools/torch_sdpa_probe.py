"""PyTorch's own SDPA at the bench shape (library reference point), for ncu."""
import torch
import torch.nn.functional as F

shp = (32, 32, 4096, 128)
q, k, v = (torch.rand(shp, device="cuda", dtype=torch.float16) * 2 - 1 for _ in range(3))
for _ in range(3):
    o = F.scaled_dot_product_attention(q, k, v)
torch.cuda.synchronize()
print("ok", o.shape)
