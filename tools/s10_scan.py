"""Developer: convergence of the S10 workload for a few cell sizes / options."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, synth
from paper_1812_05540_b200 import Tsp
for spec in sys.argv[1:]:
    kv = dict(x.split("=") for x in spec.split(",")) if spec else {}
    gen = {k: float(v) for k, v in kv.items() if k in ("length", "perm_sigma", "perm_median", "burden_perm")}
    opts = {k: (float(v) if "." in v else int(v)) for k, v in kv.items() if k not in gen}
    pb = synth.generate("S10", **gen)
    g = Tsp(pb, **opts).setup()
    x = torch.zeros(pb.n, dtype=torch.float64, device="cuda")
    info = g.solve(torch.from_numpy(pb.b).cuda(), x, max_iters=1000)
    print(spec, info["iterations"], info["status"], "%.2e" % info["true_relres"], "%.2f ms/it" % (info["t_solve_s"] * 1e3 / max(info["iterations"], 1)), flush=True)
    g.close()
