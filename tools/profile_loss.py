"""Runs the loss front end (mask + Eq. 9 loss) on a config-3-sized frame for profilers."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2402_10128_b200 as G  # noqa: E402

W, H = 1297, 840
g = torch.Generator(device="cuda").manual_seed(0)
gt = torch.rand((3, H, W), device="cuda", generator=g)
img = (gt + 0.1 * torch.randn((3, H, W), device="cuda", generator=g)).clamp(0, 1).contiguous()
loss = G.Loss(W, H)
for _ in range(3):
    m = loss.mask(gt, 0.75)
    out, dL = loss(img, gt, m)
torch.cuda.synchronize()
print(out.cpu().numpy())
