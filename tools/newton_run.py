"""A GPU-resident simulation run: per-cell fields -> device assembly -> handle -> implicit time
steps by tsp_newton_step with a BHP ramp and telescoping time steps (dt_k = min(dt_max, dt0 growth^k), halved and
retried when Newton fails).  Prints one JSON line per time step and a summary.
  python tools/newton_run.py [C5] [steps] [dt0_days] [growth]"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
from paper_1812_05540_b200 import Tsp, assemble, masses, residual  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C4"
nsteps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
dt0 = float(sys.argv[3]) * 86400.0 if len(sys.argv) > 3 else 86400.0
growth = float(sys.argv[4]) if len(sys.argv) > 4 else 2.0
dt_max = 30 * 86400.0
ramp = 2
dev = torch.device("cuda", 0)
f = synth.fields(cfg, x_rand=False)
prm = dict(f["params"])
s = synth.sizes(prm["nx"], prm["ny"], prm["nz"])
Nn = s["Nn"]
x0 = np.zeros(s["n"])
x0[3 * Nn::2] = f["sat"]
x0[3 * Nn + 1::2] = f["pres"]
ref = {k: torch.from_numpy(np.ascontiguousarray(v)).to(dev) for k, v in
       dict(E=f["E"], perm=f["perm"], phi=f["phi"], pres=f["pres"], well=f["well"]).items()}
x = torch.from_numpy(x0).to(dev)
torch.cuda.synchronize()
t0 = time.perf_counter()
ap = assemble(prm, dict(f, phi0=f["phi"]))
# NEWTON_OPTS=amg_smoother=2,local_sweeps=2 : library options of the handle (e.g. the fastest linear variant)
hopts = {k: int(v) for k, v in (kv.split("=") for kv in filter(None, os.environ.get("NEWTON_OPTS", "").split(",")))}
g = Tsp(ap, **hopts)
del ap
g.setup(1)                                   # mechanics AMG once per simulation
m0 = masses(prm, ref, x)
r_off = residual(prm, ref, x, m0, prm["dt"])[:3 * Nn].contiguous()
torch.cuda.synchronize()
t_init = time.perf_counter() - t0
print(json.dumps({"config": cfg, "dof": s["n"], "init_s": t_init, "options": hopts}), flush=True)
dbhp, t_sim, dt, tot_newton, tot_lin, t_all = prm["well_dbhp"], 0.0, dt0, 0, 0, 0.0
for step in range(nsteps):
    p_step = dict(prm, well_dbhp=dbhp * min(1.0, (step + 1) / ramp))
    for attempt in range(4):
        xs = x.clone()
        mprev = masses(p_step, ref, x)
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        info = g.newton_step(p_step, ref, x, mprev, dt, r_off=r_off)
        torch.cuda.synchronize()
        el = time.perf_counter() - t1
        if info["status"] == "OK":
            break
        x.copy_(xs)
        dt *= 0.5                                # time-step cut
    t_sim += dt
    tot_newton += info["newton_iters"]
    tot_lin += info["lin_iters"]
    t_all += el
    print(json.dumps({"step": step, "dt_days": dt / 86400, "t_days": t_sim / 86400, "status": info["status"],
                      "newton": info["newton_iters"], "fgmres": info["lin_hist"], "halvings": info["halvings"],
                      "res": [float("%.3e" % r) for r in info["res_hist"]], "s": el,
                      "s_per_newton": el / max(info["newton_iters"], 1)}), flush=True)
    dt = min(dt_max, dt * growth)
xs = x.cpu().numpy()
print(json.dumps({"summary": cfg, "steps": nsteps, "newton": tot_newton, "fgmres": tot_lin, "solve_s": t_all,
                  "max_u_m": float(np.abs(xs[:3 * Nn]).max()), "max_ds": float(np.abs(xs[3 * Nn::2] - x0[3 * Nn::2]).max()),
                  "max_dp_MPa": float(np.abs(xs[3 * Nn + 1::2] - x0[3 * Nn + 1::2]).max() / 1e6)}), flush=True)
g.close()
