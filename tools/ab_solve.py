"""Developer A/B: device time per FGMRES iteration of repeated solves at a config (CUDA events), one process.
  python tools/ab_solve.py [C5] [reps]   (environment knobs select the variant, e.g. TSP_NO_OP_FUSE=1)"""
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
print(f"{cfg} {os.environ.get('TSP_NO_OP_FUSE', 'fused')}: {info['iterations']} it, ms/iter " + " ".join(f"{m:.3f}" for m in ms),
      flush=True)
