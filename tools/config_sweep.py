"""Per-config records: for each BASELINE.json config that the oracle can run in full on the host
(C1-C4), one JSON line with the GPU path (setup + FGMRES(64) to 1e-8, device-timed, the bench's step) next to the
oracle's FULL run of the same step on the same input (its own setup and its own FGMRES to 1e-8 on one host core;
no extrapolation), and the timing-only "oracle-omp" row: the OpenMP build of the same oracle source on all host
cores (tools/oracle_run.py with ORACLE_OMP=1; row loops parallel, dot products / sweeps / setup sequential), whose x
must be bitwise the single-core run's.  Also the preconditioner apply alone, GDoF/s, and the iteration counts.
  python tools/config_sweep.py [C1 C2 C3 C4]   > profiles/r02_configs.jsonl"""
import hashlib
import json
import os
import subprocess
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
import synth  # noqa: E402
from paper_1812_05540_b200 import Tsp  # noqa: E402

cfgs = sys.argv[1:] or ["C1", "C2", "C3", "C4"]
cpu_model = next((ln.split(":", 1)[1].strip() for ln in open("/proc/cpuinfo") if ln.startswith("model name")), None)
dev = torch.device("cuda", 0)
for cfg in cfgs:
    pb = synth.generate(cfg)
    g = Tsp(pb)
    b = torch.from_numpy(pb.b).to(dev)
    x = torch.zeros(pb.n, dtype=torch.float64, device=dev)
    steps = []
    for rep in range(4):                      # 2 warm-up steps, 2 timed; setup MECH and FLOW timed apart (Table 2)
        x.zero_()
        e0, e1, e2, e3 = (torch.cuda.Event(enable_timing=True) for _ in range(4))
        e0.record()
        g.setup(1)
        e1.record()
        g.setup(2)
        e2.record()
        info = g.solve(b, x, rtol=1e-8, restart=64, max_iters=1000)
        e3.record()
        torch.cuda.synchronize()
        steps.append((e0.elapsed_time(e1), e1.elapsed_time(e2), e2.elapsed_time(e3), info))
    sm = float(np.mean([s[0] for s in steps[2:]]))
    sf = float(np.mean([s[1] for s in steps[2:]]))
    su = sm + sf
    so = float(np.mean([s[2] for s in steps[2:]]))
    fwd_gpu = float(np.linalg.norm(x.cpu().numpy() - pb.x_rand) / np.linalg.norm(pb.x_rand))
    it = steps[-1][3]["iterations"]
    z = torch.empty_like(b)
    for _ in range(3):
        g.apply_preconditioner(b, z)
    a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a0.record()
    for _ in range(20):
        g.apply_preconditioner(b, z)
    a1.record()
    torch.cuda.synchronize()
    apply_ms = a0.elapsed_time(a1) / 20
    st = g.stats()
    last = steps[-1][3]
    cyc = last["restarts"] + 2
    bytes_iter = (st["bytes_iter_base"] * it + st["bytes_operator"] * cyc + last["bytes_krylov"]) / max(it, 1)
    try:
        hbm = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")))["hbm_gbs"]
    except Exception:
        hbm = 6650.0
    H_g = [g.hierarchy(w) for w in (0, 1)]
    rng = np.random.default_rng(5)
    v_par = rng.uniform(-1, 1, pb.n)
    zt = torch.empty_like(b)
    g.apply_preconditioner(torch.from_numpy(v_par).to(dev), zt)
    z_gpu = zt.cpu().numpy()
    clk = subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm,clocks.mem,clocks_throttle_reasons.active", "--format=csv,noheader"],
                         capture_output=True, text=True).stdout.strip()
    g.close()
    # the oracle, full step on the same input
    t0 = time.perf_counter()
    o = oracle.Oracle(pb).setup()
    t1 = time.perf_counter()
    xo, io = o.solve(pb.b, rtol=1e-8, m=64)
    t2 = time.perf_counter()
    fwd_orc = float(np.linalg.norm(xo - pb.x_rand) / np.linalg.norm(pb.x_rand))
    # parity results of this record: hierarchies bitwise, one application, |delta it|
    keys = ("A_rp", "A_ci", "A_v", "dl1")
    hier_ok = all(len(H_g[w]) == o.num_levels(w) and all(
        all(np.array_equal(lo[k], lg[k]) for k in keys + (() if lo["coarsest"] else ("agg", "P_rp", "P_ci", "P_v")))
        for lo, lg in zip(o.hierarchy(w), H_g[w])) for w in (0, 1))
    z_orc = o.apply(v_par)
    apply_err = float(np.linalg.norm(z_gpu - z_orc) / np.linalg.norm(z_orc))
    nproc = os.cpu_count()
    x_sha1 = hashlib.sha1(np.ascontiguousarray(xo).tobytes()).hexdigest()
    if os.environ.get("SWEEP_NO_OMP"):       # C5: two oracle processes do not fit the host RAM; run oracle_run.py after this one
        omp = {"iterations": None, "setup_s": None, "solve_s": None, "step_s": float("nan"), "x_sha1": None}
    else:
        env = dict(os.environ, ORACLE_OMP="1", OMP_NUM_THREADS=str(nproc))
        out = subprocess.run([sys.executable, os.path.join(os.path.dirname(os.path.abspath(__file__)), "oracle_run.py"), cfg],
                             env=env, capture_output=True, text=True, check=True).stdout
        omp = json.loads(out.strip().splitlines()[-1])
    rec = {"config": cfg, "grid": [pb.nx, pb.ny, pb.nz], "dof": pb.n,
           "gpu": {"iterations": it, "setup_mech_ms": sm, "setup_flow_ms": sf, "setup_ms": su, "solve_ms": so,
                   "step_ms": su + so, "forward_error": fwd_gpu,
                   "iters_per_s": it / ((su + so) * 1e-3), "ms_per_iter": so / max(it, 1),
                   "apply_ms": apply_ms, "apply_gdof_per_s": pb.n / (apply_ms * 1e-3) / 1e9,
                   "true_relres": steps[-1][3]["true_relres"],
                   "iteration_roofline": {"bytes_per_iter": bytes_iter, "achieved_gbs": bytes_iter / (so / max(it, 1) * 1e-3) / 1e9,
                                          "peak_gbs": hbm, "frac": bytes_iter / (so / max(it, 1) * 1e-3) / 1e9 / hbm},
                   "levels": st["levels"], "clocks_sm_mem_reasons": clk},
           "parity": {"hierarchies_bit_exact": bool(hier_ok), "apply_rel_err": apply_err,
                      "delta_iterations": int(abs(io["iterations"] - it))},
           "oracle": {"iterations": io["iterations"], "status": io["status"], "setup_s": t1 - t0, "solve_s": t2 - t1,
                      "forward_error": fwd_orc, "true_relres": io["true_relres"], "cpu_model": cpu_model,
                      "host_nproc": os.cpu_count(),
                      "step_s": t2 - t0, "iters_per_s": io["iterations"] / (t2 - t0), "cores": 1,
                      "kind": "oracle (plain C, full run, no extrapolation)"},
           "oracle_omp": {"iterations": omp["iterations"], "setup_s": omp["setup_s"], "solve_s": omp["solve_s"],
                          "step_s": omp["step_s"], "cores": nproc, "cpu_model": cpu_model,
                          "bitwise_same_x": omp["x_sha1"] == x_sha1, "x_sha1_single_core": x_sha1,
                          "kind": "oracle-omp (timing only: OpenMP build of oracle.c, row loops on all cores)"},
           "speedup_step_vs_omp": omp["step_s"] / ((su + so) * 1e-3),
           "iterations_match_pm1": abs(io["iterations"] - it) <= 1,
           "speedup_step": (t2 - t0) / ((su + so) * 1e-3)}
    print(json.dumps(rec), flush=True)
