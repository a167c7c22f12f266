"""Developer: per-class live kernel times of the operator and the preconditioner at a config (CUDA events).
  python tools/kbench.py [C5] [reps]    (TSP_LIB_DEV=path/to/libtsp.so for A/B builds)"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
from paper_1812_05540_b200 import Tsp  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C5"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
pb = synth.generate(cfg)
opts = {k: int(v) for k, v in (kv.split("=") for kv in filter(None, os.environ.get("KB_OPTS", "").split(",")))}
g = Tsp(pb, **opts).setup()
v = torch.from_numpy(np.random.default_rng(1).uniform(-1, 1, pb.n)).cuda()
y = torch.empty_like(v)
for _ in range(3):
    g.apply_operator(v, y); g.apply_preconditioner(v, y)
torch.cuda.synchronize()
g.prof_enable(True)
for _ in range(reps):
    g.apply_operator(v, y)
    g.apply_preconditioner(v, y)
torch.cuda.synchronize()
p = g.prof_read()
g.prof_enable(False)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(reps):
    g.apply_operator(v, y)
e1.record(); torch.cuda.synchronize(); op_ms = e0.elapsed_time(e1) / reps
e0.record()
for _ in range(reps):
    g.apply_preconditioner(v, y)
e1.record(); torch.cuda.synchronize(); pc_ms = e0.elapsed_time(e1) / reps
print(f"[{os.environ.get('TSP_LIB_DEV', 'libtsp.so')}] {cfg}: operator {op_ms:.3f} ms, preconditioner {pc_ms:.3f} ms")
for k, d in sorted(p.items(), key=lambda kv: -kv[1]["ms"]):
    print(f"  {k:14s} {d['ms'] / d['launches'] * 1e3:9.1f} us/launch  {d['bytes'] / d['ms'] / 1e6:7.0f} GB/s  x{d['launches'] / reps:.0f}")
