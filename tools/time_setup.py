"""Developer: wall time of tsp_setup (MECH|FLOW) after warm-up; TSP_DEBUG=1 prints phase times."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, synth
from paper_1812_05540_b200 import Tsp
pb = synth.generate(sys.argv[1] if len(sys.argv) > 1 else "C5")
g = Tsp(pb)
for k in range(4):
    torch.cuda.synchronize(); t = time.time()
    g.setup()
    torch.cuda.synchronize()
    print("setup wall %.1f ms" % ((time.time() - t) * 1e3), flush=True)
