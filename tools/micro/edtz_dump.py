"""Dump the EDT pass-z input (packed (dj, di) int32 per voxel, the pass-y
output left in the workspace by ct_edt) and the distance map of the C2 t = 0
vessel channel, for tools/micro/edtz_ab.cu.  python tools/micro/edtz_dump.py DIR"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1407_2089_b200 import synth  # noqa: E402
from paper_1407_2089_b200.imaging import VoxelSpacing  # noqa: E402
from paper_1407_2089_b200.pipeline import FramePipeline  # noqa: E402

out = sys.argv[1] if len(sys.argv) > 1 else "/tmp"
spec = synth.C2
pipe = FramePipeline(spec.dims, spec.dtype, VoxelSpacing(0.8, 0.8, 1.0))
rv = synth.generate(spec, 0, synth.VESSEL)
pipe.vessel(rv)
torch.cuda.synchronize()
nx, ny, nz = spec.dims
N = nx * ny * nz
off = (N * 2 + 255) & ~255
w = pipe.ework.view(torch.uint8)
pk = w[off:off + 4 * N].view(torch.int32).cpu().numpy()
pk.tofile(os.path.join(out, "edtz_pk.bin"))
pipe.dist.cpu().numpy().astype(np.float64).tofile(os.path.join(out, "edtz_out.bin"))
pipe.vmask.cpu().numpy().tofile(os.path.join(out, "edtz_mask.bin"))
print("dumped", nx, ny, nz, "fg", float(pipe.vmask.float().mean()))
