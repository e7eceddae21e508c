"""dev probe: batched k-NN on cfg5-like descriptors (used under ncu)."""
import os as _os, sys as _sys; _sys.path.insert(0, _os.path.dirname(_os.path.dirname(_os.path.abspath(__file__))))
import sys
import time

import numpy as np

import paper_1712_06326_b200 as zb
import workloads

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 22
D = int(sys.argv[2]) if len(sys.argv) > 2 else 16
nq = int(sys.argv[3]) if len(sys.argv) > 3 else 2048
coords, queries = workloads.cfg5_descriptors(n, D, nq)
idx = zb.ZCurveIndex.from_descriptors(coords, np.arange(n, dtype=np.uint32), D)
ms, stats, _ = idx.knn_batch_bench(queries, 80, reps=1)
print(f"n={n} D={D} nq={nq} ms={ms:.3f} q/s={nq / ms * 1e3:.0f} stats={stats.tolist()} touched={stats[1] / (nq * n):.3f}")
