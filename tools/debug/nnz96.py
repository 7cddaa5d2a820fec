"""Debug: MRF nnz at nz = 96 (ct_mrf / ct_mrf_decide / ct_sign_sum vs oracle)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
from paper_1407_2089_b200 import synth, _dev
from paper_1407_2089_b200._lib import call, workspace_bytes
from oracle import oracle as O

def run(v, fn):
    nx, ny, nz = v.shape
    dv = torch.from_numpy(v).cuda()
    work = torch.empty(workspace_bytes(4, nx, ny, nz, 1), dtype=torch.uint8, device="cuda")
    state = torch.zeros(9, dtype=torch.float64, device="cuda")
    hist = torch.zeros(65536, dtype=torch.int64, device="cuda")
    call(fn, dv.data_ptr(), 1, nx, ny, nz, work.data_ptr(), state.data_ptr(), hist.data_ptr(), _dev.stream_handle())
    torch.cuda.synchronize()
    return state.cpu().numpy()

spec = synth.C4_CROP
for shape in [(1024, 1024, 96), (64, 1024, 96), (1024, 64, 96), (128, 30, 96), (1024, 1024, 64)]:
    s2 = synth.SceneSpec(*shape, "u8", n_cells=10, n_tubes=36, seed=4)
    v = synth.generate(s2, 1, synth.VESSEL).cpu().numpy()
    ss = O.sign_sum(v)
    ref = np.count_nonzero(ss)
    a = run(v, "ct_mrf"); b = run(v, "ct_mrf_decide")
    dv = torch.from_numpy(v).cuda()
    out = torch.empty(shape, dtype=torch.int64, device="cuda")
    call("ct_sign_sum", dv.data_ptr(), 1, *shape, out.data_ptr(), _dev.stream_handle())
    g = out.cpu().numpy()
    print(shape, "oracle", ref, "ct_mrf", a[3], "decide", b[3], "sign_sum kernel", np.count_nonzero(g),
          "sign arrays equal", np.array_equal(g, ss), flush=True)
    if np.count_nonzero(g) != b[3]:
        print("   decide differs by", b[3] - ref)
