"""Writes the config-3 forward image, final T and n_contrib of the loaded libges.so to a
.npz (compare two builds bit for bit: python tools/image_bits.py out.npz)."""
import os
import sys

sys.path.insert(0, os.getcwd())
import numpy as np
import torch

import ges_inputs as gi
import paper_2402_10128_b200 as G

sc = gi.make_config(int(sys.argv[2]) if len(sys.argv) > 2 else 3)
cam = sc.cameras[0]
params = G.PlanarParams.from_inputs(sc.particles)
st = G.Settings(rho=sc.rho)
r = G.Renderer(params.P, cam.width, cam.height)
img = r.forward(params, cam, st)
torch.cuda.synchronize()
W, H = cam.width, cam.height
np.savez(sys.argv[1], image=img.cpu().numpy(), T=r.frame.view("final_T", torch.float32, W * H).cpu().numpy(),
         n=r.frame.view("n_contrib", torch.int32, W * H).cpu().numpy())
