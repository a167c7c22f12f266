"""Developer: phase times of the tile-ILU kernel (k_ilu_apply2) from %globaltimer stamps in a -DTSP_ILU_TIMING
build (TSP_LIB_DEV=build_var/libtsp_ilut.so): per tile, phase 0 (step 6), forward sweep, backward sweep."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
from paper_1812_05540_b200 import Tsp, lib  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C5"
pb = synth.generate(cfg)
g = Tsp(pb).setup()
v = torch.from_numpy(np.random.default_rng(1).uniform(-1, 1, pb.n)).cuda()
z = torch.empty_like(v)
for _ in range(3):
    g.apply_preconditioner(v, z)
torch.cuda.synchronize()
L = lib()
n = 8192
buf = (C.c_ulonglong * (4 * n))()
L.tsp_dev_ilu_timers(buf, n)
t = np.frombuffer(buf, dtype=np.uint64).reshape(n, 4).astype(np.float64)
ok = t[:, 3] > 0
t = t[ok]
t0 = t[:, 0].min()
ph0, fwd, bwd, tot = t[:, 1] - t[:, 0], t[:, 2] - t[:, 1], t[:, 3] - t[:, 2], t[:, 3] - t[:, 0]
print(f"{cfg}: {ok.sum()} tiles, kernel span {(t[:, 3].max() - t0) / 1e3:.1f} us")
for name, a in (("phase0", ph0), ("forward", fwd), ("backward", bwd), ("tile", tot)):
    print(f"  {name:9s} mean {a.mean() / 1e3:7.2f} us  p10 {np.percentile(a, 10) / 1e3:7.2f}  p90 {np.percentile(a, 90) / 1e3:7.2f}")
