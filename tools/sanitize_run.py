"""Developer: a small end-to-end run for compute-sanitizer (C1 + a ragged grid; every variant once)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, synth
from paper_1812_05540_b200 import Tsp
for kw, opts in ((dict(config="C1"), {}), (dict(nx=19, ny=7, nz=21, recipe=2, perm_sigma=2.0), {}),
                 (dict(config="C1"), dict(cpr_mode=1, aps_mode=1)), (dict(config="C1"), dict(fs_mode=1))):
    cfg = kw.pop("config", None)
    pb = synth.generate(cfg, **kw)
    g = Tsp(pb, **opts).setup()
    b = torch.from_numpy(pb.b).cuda(); x = torch.zeros(pb.n, dtype=torch.float64, device="cuda")
    z = torch.empty_like(b)
    g.apply_preconditioner(b, z); g.apply_operator(b, z)
    info = g.solve(b, x, max_iters=200)
    torch.cuda.synchronize()
    print(cfg, kw, opts, info["iterations"], info["status"])
    g.close()
