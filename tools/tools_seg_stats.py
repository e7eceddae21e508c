"""Dev probe: cfg2 MSD segment-length statistics (layout + top nb Morton bytes) per depth."""
import os as _os, sys as _sys; _sys.path.insert(0, _os.path.dirname(_os.path.dirname(_os.path.abspath(__file__))))
import numpy as np
import paper_1712_06326_b200 as zb
import workloads
img, kn, p = workloads.cfg2()
mi = zb.MultiIndex(img, kn, zb.index_config(patch_size=11, dims=12))
D = 12
top = []
for l in range(8):
    coords, _ = mi.index_arrays(l)
    k = np.zeros(len(coords), dtype=np.uint64)
    for L in range(7, -1, -1):
        for d in range(D):
            pos = L * D + D - 1 - d
            if pos >= 64:
                k |= ((coords[:, d].astype(np.uint64) >> np.uint64(L)) & np.uint64(1)) << np.uint64(pos - 64)
    top.append(np.stack([np.full(len(k), l, dtype=np.uint64), k]))
for nb in (2, 3, 4):
    lens = []
    for l in range(8):
        s = top[l][1] >> np.uint64(32 - 8 * nb)
        _, c = np.unique(s, return_counts=True)
        lens.append(c)
    c = np.concatenate(lens).astype(np.float64)
    N = c.sum()
    print(f"nb={nb}: segments {len(c)}, mean {c.mean():.1f}, record-weighted mean {np.sum(c*c)/N:.1f}, "
          f"p50 {np.median(c):.0f}, p99 {np.percentile(c,99):.0f}, max {c.max():.0f}, "
          f"records in segs>64 {c[c>64].sum()/N:.3f}, >256 {c[c>256].sum()/N:.3f}")
