import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np, torch, synth
from test_gpu_multirank import _run_ranks, _work, _glue, GRID
pb = synth.generate(**GRID)
P, rep = int(sys.argv[1]), int(sys.argv[2])
one = _run_ranks(pb, 1, _work(pb), replicate_rows=rep)[0]
print("P1", one["info"])
for trial in range(2):
    many = _run_ranks(pb, P, _work(pb), replicate_rows=rep)
    parts = list(zip(many, [synth.local_problem(pb, r, P) for r in range(P)]))
    print("P", P, [m["info"] for m in many][0])
    for key in ("y", "z", "x"):
        g = _glue(parts, key, pb, P)
        d = np.abs(g - one[key])
        print(key, "maxdiff", d.max(), "n diff", (d > 0).sum(), "first", np.flatnonzero(d)[:5])
