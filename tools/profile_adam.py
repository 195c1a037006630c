"""Times the fused Adam step on a config-3-sized planar buffer (CUDA events)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2402_10128_b200 as G  # noqa: E402

P, deg = 1500000, 3
p = G.PlanarParams(torch.randn((G.n_planes(deg), P), device="cuda"), P, deg)
g = G.PlanarParams(torch.randn((G.n_planes(deg), P), device="cuda") * 1e-3, P, deg)
opt = G.Adam(p)
for _ in range(3):
    opt.step(p, g)
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(20):
    opt.step(p, g)
b.record()
b.synchronize()
ms = a.elapsed_time(b) / 20
print(f"adam {ms:.3f} ms  {28 * p.flat.numel() / ms / 1e6:.0f} GB/s")
