"""Developer: per-iteration time of repeated solves with and without the CUDA-graph iteration body."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, synth
from paper_1812_05540_b200 import Tsp
for cfg in sys.argv[1:]:
    pb = synth.generate(cfg)
    g = Tsp(pb).setup()
    b = torch.from_numpy(pb.b).cuda()
    for mode in ("eager", "graph"):
        if mode == "eager":
            os.environ["TSP_NO_GRAPH"] = "1"
        else:
            os.environ.pop("TSP_NO_GRAPH", None)
        ts = []
        for rep in range(4):
            x = torch.zeros(pb.n, dtype=torch.float64, device="cuda")
            info = g.solve(b, x, rtol=1e-8)
            ts.append(info["t_solve_s"] * 1e3 / info["iterations"])
        print(f"{cfg} {mode}: {info['iterations']} it, ms/iter per solve: " + " ".join(f"{t:.3f}" for t in ts), flush=True)
    g.close()
