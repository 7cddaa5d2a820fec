"""Vessel-channel mask statistics on C2 (how sparse the EDT sites are)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
from paper_1407_2089_b200 import synth
from paper_1407_2089_b200.imaging import VoxelSpacing
from paper_1407_2089_b200.pipeline import FramePipeline
spec = synth.C2
pipe = FramePipeline(spec.dims, spec.dtype, VoxelSpacing(0.8, 0.8, 1.0))
rv = synth.generate(spec, 0, synth.VESSEL)
res = pipe.vessel(rv)
torch.cuda.synchronize()
m = pipe.vmask
mb = m.bool()
print("fg fraction", mb.float().mean().item(), "otsu t", int(pipe.votsu[0].item()))
xl = mb.any(dim=0)  # (ny, nz): x-lines with foreground
print("x-lines with fg", xl.float().mean().item())
sites = xl.sum(dim=0).float()  # per k: number of j with an x-line site
print("sites per y-line: mean %.1f max %d" % (sites.mean().item(), int(sites.max().item())))
