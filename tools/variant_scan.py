"""Setup / second-stage variants (NEXT-f2, NEXT-f3) on one config: iterations, ms per iteration, setup, step."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, synth
from paper_1812_05540_b200 import Tsp
cfg = sys.argv[1] if len(sys.argv) > 1 else "C5"
VARIANTS = [
    ("default (quasi-IMPES, full A_ps, K_dr, ILU x1)", {}),
    ("true-IMPES", dict(cpr_mode=1)),
    ("diagonal A_ps", dict(aps_mode=1)),
    ("fs_modulus_scale 1.8 (uniaxial)", dict(fs_modulus_scale=1.8)),
    ("RSL, 2 Richardson steps", dict(fs_mode=1, rsl_iters=2)),
    ("hbgs x1", dict(second_stage=1, local_sweeps=1)),
    ("hbgs x3 (staircase M_L)", dict(second_stage=1, local_sweeps=3)),
    ("ILU x2", dict(local_sweeps=2)),
    ("ILU x2 + modulus 1.8 + diagonal A_ps", dict(local_sweeps=2, fs_modulus_scale=1.8, aps_mode=1)),
    ("GS AMG smoothers (P:711)", dict(amg_smoother=1)),
    ("GS AMG smoothers + hbgs x3 (the paper's staircase settings)", dict(amg_smoother=1, second_stage=1, local_sweeps=3)),
    ("GS AMG smoothers + ILU x2", dict(amg_smoother=1, local_sweeps=2)),
    ("Chebyshev(2) AMG smoothers", dict(amg_smoother=2)),
    ("Chebyshev(3) AMG smoothers", dict(amg_smoother=2, amg_cheb_degree=3)),
    ("Chebyshev(2) on [0.1, 1]", dict(amg_smoother=2, amg_cheb_lower=0.1)),
    ("Chebyshev(2) AMG smoothers + ILU x2", dict(amg_smoother=2, local_sweeps=2)),
    ("Chebyshev(2) pressure AMG only", dict(amg_smoother=0, amg_smoother_p=2)),
    ("Chebyshev(2) pressure AMG only + ILU x2", dict(amg_smoother=0, amg_smoother_p=2, local_sweeps=2)),
    ("Chebyshev(3) pressure AMG only", dict(amg_smoother=0, amg_smoother_p=2, amg_cheb_degree=3)),
    ("Chebyshev(2) mechanics AMG only", dict(amg_smoother=2, amg_smoother_p=0)),
    ("Chebyshev(2) mechanics AMG only + ILU x2", dict(amg_smoother=2, amg_smoother_p=0, local_sweeps=2)),
    ("Chebyshev(3) mechanics AMG only", dict(amg_smoother=2, amg_smoother_p=0, amg_cheb_degree=3)),
    ("Chebyshev(2) [0.1,1] mechanics AMG only", dict(amg_smoother=2, amg_smoother_p=0, amg_cheb_lower=0.1)),
    ("Chebyshev(2) mechanics AMG only + modulus 1.8", dict(amg_smoother=2, amg_smoother_p=0, fs_modulus_scale=1.8)),
]
if len(sys.argv) > 2:   # only the variants whose name contains this word
    VARIANTS = [v for v in VARIANTS if sys.argv[2] in v[0]]
pb = synth.generate(cfg)
b = torch.from_numpy(pb.b).cuda()
for name, opts in VARIANTS:
    g = Tsp(pb, **opts)
    g.setup()                                   # warm the allocator
    torch.cuda.synchronize(); t = time.time(); g.setup(); torch.cuda.synchronize(); ts = time.time() - t
    x = torch.zeros(pb.n, dtype=torch.float64, device="cuda")
    info = g.solve(b, x, rtol=1e-8, max_iters=1000)
    it = info["iterations"]; tsolve = info["t_solve_s"]
    print(f"| {name} | {it}{'' if info['status'] == 'OK' else ' (not converged)'} | {1e3 * tsolve / max(it, 1):.2f} | "
          f"{1e3 * ts:.0f} | {1e3 * (ts + tsolve):.0f} |", flush=True)
    g.close()
