"""Dev: distribution of the Morton key bytes of a config's layout indices (how many distinct
values the top bytes take, and how much mass the most frequent ones hold)."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1712_06326_b200 as zb
import workloads

name = sys.argv[1] if len(sys.argv) > 1 else "cfg4"
img, known, kw = getattr(workloads, name)()
mi = zb.MultiIndex(img, known, zb.index_config(**kw))
D = mi.dims
for l in range(8):
    c, _ = mi.index_arrays(l)
    n = c.shape[0]
    # Morton byte b (D = 8): bit b of every dim, dim 0 at the top
    by = []
    for b in range(8):
        v = np.zeros(n, np.uint32)
        for d in range(D):
            v |= ((c[:, d] >> b) & 1).astype(np.uint32) << (D - 1 - d)
        by.append(v)
    line = [f"layout {l}:"]
    for b in range(7, -1, -1):
        h = np.bincount(by[b], minlength=1 << D)
        nz = int((h > 0).sum())
        top = np.sort(h)[::-1]
        line.append(f"b{b}: {nz} distinct, top1 {top[0] / n:.3f}, 99.9% in {int(np.searchsorted(np.cumsum(top), 0.999 * n)) + 1}")
    print("  ".join(line))
    for depth in (2, 3, 4):
        if D != 8:
            break
        comb = np.zeros(n, np.uint64)
        for b in range(7, 7 - depth, -1):
            comb = (comb << np.uint64(8)) | by[b].astype(np.uint64)
        u, cnt = np.unique(comb, return_counts=True)
        top = np.sort(cnt)[::-1]
        print(f"   top {depth} bytes: {len(u)} distinct, 99.9% in {int(np.searchsorted(np.cumsum(top), 0.999 * n)) + 1}, largest {top[0] / n:.4f}")
