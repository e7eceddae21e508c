"""Dev probe: per-kernel device time of the cfg2/cfg4 builds (tensor-core projection vs fp64)."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1712_06326_b200 as zb
import workloads

name = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
img, known, kw = getattr(workloads, name)()
ctx = zb.Context.default()
mi = zb.MultiIndex(img, known, zb.index_config(**kw))
for _ in range(3):
    mi.rebuild()
ctx.set_profiling(True)
for _ in range(5):
    mi.rebuild()
ctx.synchronize()
prof = ctx.profile()
tot = sum(v[0] for v in prof.values())
for k, (ms, cnt) in sorted(prof.items(), key=lambda x: -x[1][0]):
    print(f"{k:32s} {ms / 5:8.3f} ms/build  {cnt // 5} launches")
print(f"{'total':32s} {tot / 5:8.3f}")
