"""Debug: repeat ct_mrf / ct_mrf_decide nnz on the C4-crop vessel frame."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
from paper_1407_2089_b200 import synth, _dev
from paper_1407_2089_b200._lib import call, workspace_bytes

def run(v, fn, dv=None):
    nx, ny, nz = v.shape
    dv = torch.from_numpy(v).cuda() if dv is None else dv
    work = torch.empty(workspace_bytes(4, nx, ny, nz, 1), dtype=torch.uint8, device="cuda")
    state = torch.zeros(9, dtype=torch.float64, device="cuda")
    hist = torch.zeros(65536, dtype=torch.int64, device="cuda")
    call(fn, dv.data_ptr(), 1, nx, ny, nz, work.data_ptr(), state.data_ptr(), hist.data_ptr(), _dev.stream_handle())
    torch.cuda.synchronize()
    return state.cpu().numpy()
shape = tuple(int(x) for x in sys.argv[1:4]) if len(sys.argv) > 3 else (1024, 1024, 96)
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 20
s2 = synth.SceneSpec(*shape, "u8", n_cells=10, n_tubes=36, seed=4)
v = synth.generate(s2, 1, synth.VESSEL).cpu().numpy()
for fn in ("ct_mrf", "ct_mrf_decide"):
    vals = [run(v, fn)[3] for _ in range(reps)]
    print(shape, fn, sorted(set(vals)), flush=True)
