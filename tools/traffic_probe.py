"""One launch of every bench kernel at its BASELINE shape (eager, through
the public launchers), in a fixed order, for ncu metric collection:

    ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_srcunit_tex_op_write.sum,\
gpu__time_duration.sum --clock-control none --csv --log-file X python tools/traffic_probe.py

tools/make_traffic.py turns the CSV into profiles/traffic.json."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2507_11978_b200 import backend as B  # noqa: E402

dev = "cuda:0"
f16, f32 = torch.float16, torch.float32


def U(shape, dt=f16):
    return (torch.rand(shape, device=dev) * 2 - 1).to(dt)


ORDER = []


def run(key, fn):
    torch.cuda.synchronize()
    ORDER.append(key)
    fn()
    torch.cuda.synchronize()


x = U((4096, 4096)); w = U((4096,)); y = torch.empty_like(x)
run("softmax", lambda: B.softmax_launch(x, y, 4096))
run("rms_norm", lambda: B.rms_norm_launch(x, w, y, 4096))
for n, key in ((1 << 20, "add_2^20"), (1 << 24, "add_2^24")):
    a, b = U((n,), f32), U((n,), f32)
    o = torch.empty_like(a)
    run(key, lambda: B.add_launch(a, b, o, 1024))
a = U((1 << 24,)); o = torch.empty_like(a)
run("silu_2^24", lambda: B.silu_launch(a, o, 1024))
A, Bm, Cm, Dm = U((4096, 4096)), U((4096, 4096)), torch.empty((4096, 4096), device=dev, dtype=f16), U((4096, 4096))
run("mm", lambda: B.mm_launch(A, Bm, Cm, 128, 128, 64))
run("addmm", lambda: B.addmm_launch(Dm, A, Bm, -0.134, -0.201, Cm, 128, 128, 64))
del A, Bm, Cm, Dm
a3, b3 = U((64, 1024, 1024)), U((64, 1024, 1024)); c3 = torch.empty_like(a3)
run("bmm", lambda: B.bmm_launch(a3, b3, c3, 128, 128, 64))
del a3, b3, c3
A, Bm = U((4096, 4096), f32), U((4096, 4096), f32); Cm = torch.empty_like(A)
run("mm_f32", lambda: B.mm_launch(A, Bm, Cm, 128, 128, 64))
del A, Bm, Cm
a3, b3 = U((64, 1024, 1024), f32), U((64, 1024, 1024), f32); c3 = torch.empty_like(a3)
run("bmm_f32", lambda: B.bmm_launch(a3, b3, c3, 128, 128, 64))
del a3, b3, c3
xc, wc = U((64, 256, 56, 56)), U((256, 256, 3, 3)); yc = torch.empty((64, 256, 54, 54), device=dev, dtype=f16)
run("conv2d", lambda: B.conv2d_launch(xc, wc, yc, 128, 128, 64))
xc, wc = xc.float(), wc.float(); yc = yc.float()
run("conv2d_f32", lambda: B.conv2d_launch(xc, wc, yc, 128, 128, 64))
del xc, wc, yc
q, k, v = (U((32, 32, 4096, 128)) for _ in range(3)); o = torch.empty_like(q)
run("sdpa", lambda: B.sdpa_launch(q, k, v, o, 128, 128))
del q, k, v, o
xs = U((32, 4096, 32, 128)); ang = torch.rand((4096, 64), device=dev) * 6 - 3
sn, cs = torch.sin(ang).half(), torch.cos(ang).half(); xo = torch.empty_like(xs)
run("rope", lambda: B.rope_launch(xs, sn, cs, xo, 64))
qs, ks, vs = xs, U((32, 4096, 32, 128)), U((32, 4096, 32, 128))
o = torch.empty((32, 32, 4096, 128), device=dev, dtype=f16)
T = lambda t: t.transpose(1, 2)  # noqa: E731
run("sdpa_rope", lambda: B.sdpa_rope_launch(T(qs), T(ks), T(vs), sn, cs, sn, cs, o, 128, 128))
print(",".join(ORDER))
