"""Developer: FGMRES restart length against iterations and time to solution at one config (device-timed solve after
one warm-up solve per m; setup excluded).  SPEC's restart is 200, R-krylov's default 64 (D9).
  python tools/restart_scan.py [C5] [m ...]   (NEWTON-style options: SCAN_OPTS=amg_smoother=2,local_sweeps=2)"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import synth  # noqa: E402
from paper_1812_05540_b200 import Tsp  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C5"
ms = [int(a) for a in sys.argv[2:]] or [32, 64, 96, 120]
opts = {k: (float(v) if "." in v else int(v)) for k, v in
        (kv.split("=") for kv in filter(None, os.environ.get("SCAN_OPTS", "").split(",")))}
pb = synth.generate(cfg)
g = Tsp(pb, **opts).setup()
b = torch.from_numpy(pb.b).cuda()
x = torch.zeros(pb.n, dtype=torch.float64, device="cuda")
for m in ms:
    g.solve(b, x, rtol=1e-8, restart=m, max_iters=2000)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    info = g.solve(b, x, rtol=1e-8, restart=m, max_iters=2000)
    e1.record()
    torch.cuda.synchronize()
    ms_ = e0.elapsed_time(e1)
    print(json.dumps({"config": cfg, "options": opts, "restart": m, "iterations": info["iterations"],
                      "status": info["status"], "solve_s": ms_ / 1e3, "ms_per_iter": ms_ / max(info["iterations"], 1),
                      "true_relres": info["true_relres"]}), flush=True)
