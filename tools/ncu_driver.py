"""Dev driver for ncu captures: one build of a config (after a warm-up build), a few fill-loop
queries and brute-force scans, so `ncu -k regex:... -c N` sees the kernels of a real step.

  python tools/ncu_driver.py cfg4 [--queries 8]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_1712_06326_b200 as zb  # noqa: E402
import workloads  # noqa: E402
from tests.helpers import fillfront  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg4"
nq = int(sys.argv[sys.argv.index("--queries") + 1]) if "--queries" in sys.argv else 8
img, kn, p = getattr(workloads, cfg)()
mi = zb.MultiIndex(img, kn, zb.index_config(**p))
mi.rebuild()
K = p["patch_size"]
front = fillfront(kn)
C = 1 if img.ndim == 2 else img.shape[2]
for i in range(nq):
    x, y = front[(i * 7919) % len(front)]
    r = K // 2
    tv = np.zeros((K, K) + img.shape[2:], np.uint8)
    tk = np.zeros((K, K), np.uint8)
    for dy in range(K):
        for dx in range(K):
            yy, xx = y - r + dy, x - r + dx
            if 0 <= yy < img.shape[0] and 0 <= xx < img.shape[1] and kn[yy, xx]:
                tv[dy, dx] = img[yy, xx]
                tk[dy, dx] = 1
    mi.query_best_patch(tv.reshape(-1), tk.reshape(-1))
    mi.brute_force_best(tv.reshape(-1), tk.reshape(-1))
print("ncu driver done", cfg, mi.n)
