"""Dev probe: phase timings of the fill loop's one-launch query (k_query_one, ZI_DEBUG_QUERY).

  python tools/query_phases.py cfg2|cfg4 [max_queries]

Runs the config's fill loop with ZI_DEBUG_QUERY=1 (each query synchronises and reads back the
%globaltimer stamps of CTA 0 and of the merging CTA) and prints median / p90 microseconds per
phase plus the candidate counts.  Phases (k_query.cu ZI_TPHASE): 1 stage + select_index +
make_query, 2 local seed, 3 bbox-pruned scan, 4 local top-k + costing, 6 merge start (last CTA),
7 compaction, 8 global k-th, 9 winner published.
"""
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

if len(sys.argv) > 1 and sys.argv[1] == "--child":
    sys.path.insert(0, ROOT)
    import paper_1712_06326_b200 as zb
    import workloads
    img, kn, p = getattr(workloads, sys.argv[2])()
    mi = zb.MultiIndex(img, kn, zb.index_config(**p))
    mi.inpaint()
    sys.exit(0)

import numpy as np  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
limit = int(sys.argv[2]) if len(sys.argv) > 2 else 10 ** 9
env = dict(os.environ, ZI_DEBUG_QUERY="1")
r = subprocess.run([sys.executable, __file__, "--child", cfg], env=env, capture_output=True, text=True)
rows = []
pat = re.compile(r"query lid=(\d+) bound_dist=(\d+) total=(\d+) m=(\d+) count=(\d+) overflow=(\d+) phases_us:(.*)")
for line in r.stderr.splitlines():
    m = pat.match(line)
    if m:
        ph = [float(x) for x in m.group(7).split()]
        rows.append([int(m.group(i)) for i in range(1, 7)] + ph)
    if len(rows) >= limit:
        break
a = np.array(rows)
print(f"{cfg}: {len(a)} queries")
names = ["lid", "bound", "total", "m", "count", "overflow"]
for i, nm in enumerate(names[1:], start=1):
    print(f"  {nm:>9}: median {np.median(a[:, i]):.0f}  p90 {np.percentile(a[:, i], 90):.0f}  max {a[:, i].max():.0f}")
labels = {1: "make_query", 2: "seed", 3: "scan", 4: "local_topk+cost", 5: "-", 6: "merge_start", 7: "compact",
          8: "kth", 9: "published"}
for j in range(9):
    col = a[:, 6 + j]
    print(f"  phase {j + 1} {labels[j + 1]:>16}: median {np.median(col):7.1f} us  p90 {np.percentile(col, 90):7.1f}")
sp = re.compile(r"qlat ctas=(\d+) start_spread_us=([\d.]+) finish_first_us=([\d.]+) finish_last_us=([\d.]+) "
                r"max_surv=(\d+) max_cand=(\d+) last_surv=(\d+) last_cand=(\d+)")
rows = [tuple(float(x) for x in m.groups()) for m in (sp.match(l) for l in r.stderr.splitlines()) if m][:limit]
if rows:
    a = np.array(rows)
    print(f"  CTAs {int(a[0, 0])}: start spread median {np.median(a[:, 1]):.1f} us, first finish {np.median(a[:, 2]):.1f}, "
          f"last finish {np.median(a[:, 3]):.1f} (p90 {np.percentile(a[:, 3], 90):.1f})")
    print(f"  survivors per CTA: max median {np.median(a[:, 4]):.0f}, candidates max median {np.median(a[:, 5]):.0f}; "
          f"the last CTA: survivors {np.median(a[:, 6]):.0f}, candidates {np.median(a[:, 7]):.0f}")
