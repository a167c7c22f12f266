"""Developer A/B: device time per FGMRES iteration of repeated solves at a config (CUDA events), one process.
  python tools/ab_solve.py [C5] [reps]   (environment knobs select the variant, e.g. TSP_NO_OP_FUSE=1; prints a digest of x for bitwise A/B)"""
import hashlib
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import synth  # noqa: E402
from paper_1812_05540_b200 import Tsp  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C5"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
pb = synth.generate(cfg)
g = Tsp(pb).setup()
b = torch.from_numpy(pb.b).cuda()
x = torch.zeros(pb.n, dtype=torch.float64, device="cuda")
g.solve(b, x)
ms = []
for _ in range(reps):
    x.zero_()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    info = g.solve(b, x)
    e1.record()
    torch.cuda.synchronize()
    ms.append(e0.elapsed_time(e1) / info["iterations"])
knobs = ",".join(f"{k}={v}" for k, v in sorted(os.environ.items()) if k.startswith("TSP_")) or "default"
digest = hashlib.sha1(x.cpu().numpy().tobytes()).hexdigest()[:12]
print(f"{cfg} {knobs}: {info['iterations']} it, x sha1 {digest}, ms/iter " + " ".join(f"{m:.3f}" for m in ms), flush=True)
