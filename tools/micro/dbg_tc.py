import sys, numpy as np, torch
sys.path.insert(0, '/root/repo/tests'); sys.path.insert(0, '/root/repo')
from test_gpu_parity import _q_exact_and_fast, _k1_path, ANISO
_k1_path(2)
for sigma, shape in [(1.0, (64, 32, 32)), (2.0, (64, 32, 64)), (3.0, (200, 64, 32)), (6.0, (64, 32, 32)), (3.0, (64, 32, 32)), (3.0, (128, 64, 64)), (4.0, (128, 64, 64)), (5.0, (128, 64, 64)), (3.0, (256, 256, 32))]:
    rng = np.random.default_rng(1)
    raw = torch.from_numpy(rng.integers(0, 256, size=shape, dtype=np.uint8)).cuda()
    q1, q2, fx = _q_exact_and_fast(raw, ANISO, sigma)
    d = (q1.int() - q2.int())
    print(sigma, shape, 'differ', int((d != 0).sum()), 'mean diff', float(d.float().mean()), 'fix', fx)
