"""Dev probe: the cfg5 vector-index build (device-resident fp32 rows) with per-kernel device time;
`python tools/vec_probe.py [log2 n] [D]`.  Rows: x = Q diag(0.9^(k/2)) z, seeded, dim 125."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1712_06326_b200 as zb  # noqa: E402

lg = int(sys.argv[1]) if len(sys.argv) > 1 else 24
D = int(sys.argv[2]) if len(sys.argv) > 2 else 16
n, dim = 1 << lg, 125
dev = torch.device("cuda", 0)
rng = np.random.default_rng(5)
Q, _ = np.linalg.qr(rng.normal(size=(dim, dim)))
scale = torch.tensor(0.9 ** (np.arange(dim) / 2.0), dtype=torch.float32, device=dev)
g = torch.Generator(device=dev).manual_seed(5)
X = torch.empty((n, dim), dtype=torch.float32, device=dev)
Qt = torch.tensor(Q.T, dtype=torch.float32, device=dev)
for b in range(0, n, 1 << 22):
    z = torch.randn((min(1 << 22, n - b), dim), generator=g, dtype=torch.float32, device=dev) * scale
    X[b:b + z.shape[0]] = z @ Qt
torch.cuda.synchronize()
ctx = zb.Context.default()
zb.VectorIndex(X, D, ctx=ctx)
ctx.set_profiling(True)
for _ in range(3):
    vi = zb.VectorIndex(X, D, ctx=ctx)
prof = ctx.profile()
for k, (ms, cnt) in sorted(prof.items(), key=lambda x: -x[1][0]):
    if cnt:
        print(f"{k:28s} {ms / 3:8.3f} ms/build")
