"""dev probe: cfg2 build step time with / without the L2 flush and per-kernel profiling events."""
import os as _os, sys as _sys; _sys.path.insert(0, _os.path.dirname(_os.path.dirname(_os.path.abspath(__file__))))
import time
import paper_1712_06326_b200 as zb
import workloads

img, known, kw = workloads.cfg2()
ctx = zb.Context.default()
mi = zb.MultiIndex(img, known, zb.index_config(**kw))
for _ in range(3):
    mi.rebuild()
for flush in (False, True):
    for prof in (False, True):
        ctx.set_profiling(prof)
        ms = []
        for _ in range(10):
            if flush:
                ctx.flush_l2()
            ctx.synchronize()
            t = time.perf_counter()
            ctx.timer_start()
            mi.rebuild()
            ms.append(ctx.timer_stop())
            wall = (time.perf_counter() - t) * 1e3
        ctx.set_profiling(False)
        print(f"flush={flush} profiling={prof}: device {sum(ms)/len(ms):.3f} ms (min {min(ms):.3f}), last wall {wall:.3f} ms")
