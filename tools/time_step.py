"""Developer: wall time of setup and solve in the bench's step loop (setup + FGMRES)."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, synth
from paper_1812_05540_b200 import Tsp
pb = synth.generate(sys.argv[1] if len(sys.argv) > 1 else "C5")
g = Tsp(pb)
if os.environ.get("PROF"): g.prof_enable(True)
b = torch.from_numpy(pb.b).cuda(); x = torch.zeros(pb.n, dtype=torch.float64, device="cuda")
for k in range(4):
    torch.cuda.synchronize(); t0 = time.time()
    g.setup()
    torch.cuda.synchronize(); t1 = time.time()
    info = g.solve(b, x, rtol=1e-8, restart=64, max_iters=int(sys.argv[2]) if len(sys.argv) > 2 else 1000)
    torch.cuda.synchronize(); t2 = time.time()
    print("setup %.1f ms  solve %.1f ms (library %.1f ms, %d it)" % ((t1 - t0) * 1e3, (t2 - t1) * 1e3, info["t_solve_s"] * 1e3,
                                                                   info["iterations"]), flush=True)
