"""The oracle's full step (setup + FGMRES(64) to 1e-8) on one config, one JSON line: timings, iterations and a
digest of x.  tools/config_sweep.py runs it with ORACLE_OMP=1 for the timing-only "oracle-omp" row (the OpenMP
build of oracle.c: row-independent loops on all host cores, bitwise the same x as the plain build).
  ORACLE_OMP=1 python tools/oracle_run.py C2 ['{"amg_smoother": 2}']"""
import hashlib
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402
import synth  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C1"
opts = json.loads(sys.argv[2]) if len(sys.argv) > 2 else {}
pb = synth.generate(cfg)
t0 = time.perf_counter()
o = oracle.Oracle(pb, **opts).setup()
t1 = time.perf_counter()
x, info = o.solve(pb.b, rtol=1e-8, m=64)
t2 = time.perf_counter()
print(json.dumps({"config": cfg, "omp": os.environ.get("ORACLE_OMP", "0"), "threads": os.environ.get("OMP_NUM_THREADS"),
                  "iterations": info["iterations"], "setup_s": t1 - t0, "solve_s": t2 - t1, "step_s": t2 - t0,
                  "x_sha1": hashlib.sha1(x.tobytes()).hexdigest(),
                  "oracle_lib": next((ln.split()[-1] for ln in open("/proc/self/maps") if "liboracle" in ln), None)}), flush=True)
