"""Developer: a small end-to-end run for compute-sanitizer (C1 + a ragged grid; every variant and entry point once:
setup variants, the three AMG smoothers, both second stages, two sweeps, value update + frozen-aggregation refresh,
FGMRES with and without the bulk-copy pass, the DCGS2 fallback, Richardson, device assembly)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, synth
from paper_1812_05540_b200 import Tsp, assemble
RAG = dict(nx=19, ny=7, nz=21, recipe=2, perm_sigma=2.0)
RUNS = ((dict(config="C1"), {}), (dict(RAG), {}),
        (dict(config="C1"), dict(cpr_mode=1, aps_mode=1)), (dict(config="C1"), dict(fs_mode=1)),
        (dict(RAG), dict(amg_smoother=1)), (dict(RAG), dict(amg_smoother=2, local_sweeps=2)),
        (dict(RAG), dict(second_stage=1)), (dict(config="C1"), dict(amg_smoother=2, amg_smoother_p=0, amg_cheb_lower=0.1)))
for kw, opts in RUNS:
    cfg = kw.pop("config", None)
    pb = synth.generate(cfg, **kw)
    g = Tsp(pb, **opts).setup()
    b = torch.from_numpy(pb.b).cuda(); x = torch.zeros(pb.n, dtype=torch.float64, device="cuda")
    z = torch.empty_like(b)
    g.apply_preconditioner(b, z); g.apply_operator(b, z)
    info = g.solve(b, x, max_iters=200)
    g.update_values(pb); g.setup_flow(refresh=True)
    i2 = g.solve(b, x, max_iters=200, restart=7)
    ir = g.richardson(b, x, rtol=1e-30, max_iters=3)
    torch.cuda.synchronize()
    print(cfg, kw, opts, info["iterations"], info["status"], i2["iterations"], ir["iterations"])
    g.close()
for knob in ("TSP_NO_TMA", "TSP_DCGS2_FALLBACK", "TSP_NO_GRAPH", "TSP_NO_OP_FUSE"):
    os.environ[knob] = "1"
    pb = synth.generate(None, **RAG)
    g = Tsp(pb).setup()
    b = torch.from_numpy(pb.b).cuda(); x = torch.zeros(pb.n, dtype=torch.float64, device="cuda")
    print(knob, g.solve(b, x)["iterations"])
    g.close()
    del os.environ[knob]
f = synth.fields("C1", x_rand=False)
ap = assemble(f["params"], f)
torch.cuda.synchronize()
print("assembly ok", float(ap.uu_val.abs().max()))
