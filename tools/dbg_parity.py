"""Developer diagnostics: per-field apply errors vs the oracle, and NaN hunting."""
import sys, time
import numpy as np, torch
import synth, oracle
from paper_1812_05540_b200 import Tsp

def cu(x): return torch.from_numpy(np.ascontiguousarray(x)).cuda()

cfg = sys.argv[1]
pb = synth.generate(cfg)
t = time.time(); g = Tsp(pb).setup(); torch.cuda.synchronize(); print("gpu setup", time.time() - t, g.stats()["rows"])
nu = 3 * pb.Nn
z = torch.empty(pb.n, dtype=torch.float64, device="cuda")
g.apply_preconditioner(cu(pb.b), z); torch.cuda.synchronize()
zg = z.cpu().numpy()
print("nan in z:", np.isnan(zg).sum(), "u", np.isnan(zg[:nu]).sum(), "s", np.isnan(zg[nu::2]).sum(), "p", np.isnan(zg[nu+1::2]).sum())
if len(sys.argv) > 2:
    o = oracle.Oracle(pb).setup()
    rng = np.random.default_rng(12)
    for v in (pb.b, rng.uniform(-1, 1, pb.n), rng.standard_normal(pb.n)):
      g.apply_preconditioner(cu(v), z); torch.cuda.synchronize(); zg = z.cpu().numpy()
      ref = o.apply(v)
      for nm, sl in (("u", slice(0, nu)), ("s", slice(nu, None, 2)), ("p", slice(nu + 1, None, 2)), ("all", slice(None))):
          print(nm, np.linalg.norm(zg[sl] - ref[sl]) / np.linalg.norm(ref[sl]))
    Ho, Hg = o.hierarchy(1), g.hierarchy(1)
    print("pres levels", [L["n"] for L in Ho], [L["n"] for L in Hg])
    Ho, Hg = o.hierarchy(0), g.hierarchy(0)
    print("mech levels", [L["n"] for L in Ho], [L["n"] for L in Hg])
for w in (0, 1):
    for l, L in enumerate(g.hierarchy(w)):
        print(w, l, L["n"], L["nnz"], L["coarsest"], "nan A", np.isnan(L["A_v"]).sum(), "min dl1", L["dl1"].min())
