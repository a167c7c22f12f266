import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np, torch, synth
from test_gpu_multirank import _run_ranks, _glue, GRID
pb = synth.generate(**GRID)
P, rep = int(sys.argv[1]), int(sys.argv[2])
def work_maker(maxit, what):
    def work(r, g, lp):
        g.setup()
        b = lp.local(pb.b, pb.Nn) if g.n != pb.n else pb.b
        db = torch.from_numpy(np.ascontiguousarray(b)).cuda()
        x = torch.zeros_like(db)
        if what == "solve":
            g.solve(db, x, max_iters=maxit, restart=int(os.environ.get("RST", "64")))
        else:   # apply twice in a row on the same vector, second result
            z = torch.empty_like(db)
            for _ in range(maxit): g.apply_preconditioner(db, z)
            x = z
        torch.cuda.synchronize()
        return dict(x=x.cpu().numpy())
    return work
for what in ("apply", "solve"):
    for maxit in ((1, 2, 3) if what == "apply" else (5, 8, 9, 10, 12, 16, 24, 32)):
        one = _run_ranks(pb, 1, work_maker(maxit, what), replicate_rows=rep)[0]
        many = _run_ranks(pb, P, work_maker(maxit, what), replicate_rows=rep)
        parts = list(zip(many, [synth.local_problem(pb, r, P) for r in range(P)]))
        g = _glue(parts, "x", pb, P)
        d = np.abs(g - one["x"])
        print(what, maxit, "maxdiff", d.max(), "ndiff", (d > 0).sum(), np.flatnonzero(d)[:4])
