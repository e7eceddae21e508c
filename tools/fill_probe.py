import os, sys, time
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import paper_1712_06326_b200 as zb, workloads
cfg = sys.argv[1]
img, kn, p = getattr(workloads, cfg)()
mi = zb.MultiIndex(img, kn, zb.index_config(**p))
for r in range(2):
    t = time.perf_counter(); out = mi.inpaint(); dt = time.perf_counter() - t
    print(cfg, "run", r, "seconds", dt, flush=True)
