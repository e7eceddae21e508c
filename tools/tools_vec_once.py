"""Dev probe: one cfg5 vector-index build from device-resident rows (for ncu captures)."""
import os as _os, sys as _sys; _sys.path.insert(0, _os.path.dirname(_os.path.dirname(_os.path.abspath(__file__))))
import numpy as np
import torch
import paper_1712_06326_b200 as zb
n, dim = 1 << 22, 125
g = torch.Generator(device="cuda").manual_seed(5)
X = torch.randn((n, dim), generator=g, device="cuda", dtype=torch.float32)
vi = zb.VectorIndex(X, 16)
vi = zb.VectorIndex(X, 16)
print("build ms", vi.build_ms)
