"""Developer: convergence of the GPU solver on configs / restart lengths."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import synth
from paper_1812_05540_b200 import Tsp
for spec in sys.argv[1:]:
    cfg, *kv = spec.split(",")
    kw = {k: float(v) if "." in v or "e" in v else int(v) for k, v in (x.split("=") for x in kv)}
    restart = int(kw.pop("restart", 64))
    pb = synth.generate(cfg, **kw)
    g = Tsp(pb).setup()
    b = torch.from_numpy(pb.b).cuda(); x = torch.zeros(pb.n, dtype=torch.float64, device="cuda")
    for maxit in (50, 100, 200, 400, 1000):
        t = time.time(); info = g.solve(b, x, max_iters=maxit, restart=restart)
        print(spec, maxit, info["iterations"], "%.2e" % info["true_relres"], "%.2fs" % (time.time() - t), flush=True)
        if info["status"] == "OK": break
    g.close()
