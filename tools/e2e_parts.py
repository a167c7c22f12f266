"""Developer: wall-time parts of the end-to-end step from host fields (bench.py e2e_gpu_assembly): H2D of the fields,
tsp_assemble, tsp_create from device blocks, b = A x_rand, setup, solve, D2H, destroy.
  python tools/e2e_parts.py [C5]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
from paper_1812_05540_b200 import Tsp, assemble  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C5"
dev = torch.device("cuda", 0)
fl = synth.fields(cfg)
hf = {k: torch.from_numpy(np.ascontiguousarray(fl[k])).pin_memory() for k in ("E", "perm", "phi", "sat", "pres", "well", "x_rand")}
n = len(fl["x_rand"])
xh = torch.zeros(n, dtype=torch.float64).pin_memory()


def t():
    torch.cuda.synchronize()
    return time.perf_counter()


for rep in range(3):
    T = [t()]
    d = {k: v.to(dev, non_blocking=True) for k, v in hf.items()}
    T.append(t())
    ap = assemble(fl["params"], d)
    T.append(t())
    h = Tsp(ap)
    T.append(t())
    del ap
    b = torch.empty(n, dtype=torch.float64, device=dev)
    h.apply_operator(d["x_rand"], b)
    T.append(t())
    h.setup()
    T.append(t())
    x = torch.zeros(n, dtype=torch.float64, device=dev)
    info = h.solve(b, x)
    T.append(t())
    xh.copy_(x, non_blocking=True)
    T.append(t())
    h.close()
    T.append(t())
    names = ["h2d", "assemble", "create", "b=Ax", "setup", "solve", "d2h", "destroy"]
    print(cfg, rep, " ".join(f"{nm} {1e3 * (T[i + 1] - T[i]):.1f}" for i, nm in enumerate(names)), f"it {info['iterations']}",
          flush=True)
