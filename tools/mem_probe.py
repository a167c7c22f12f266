"""Developer: device memory in use after create / setup / solve (C5 by default)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, synth
from paper_1812_05540_b200 import Tsp
def used():
    f, t = torch.cuda.mem_get_info(); return (t - f) / 1e9
pb = synth.generate(sys.argv[1] if len(sys.argv) > 1 else "C5")
print("inputs on host; device used %.1f GB" % used())
g = Tsp(pb); torch.cuda.synchronize(); print("after create %.1f GB" % used())
g.setup(); torch.cuda.synchronize(); print("after setup %.1f GB" % used())
b = torch.from_numpy(pb.b).cuda(); x = torch.zeros(pb.n, dtype=torch.float64, device="cuda")
g.solve(b, x, max_iters=5); torch.cuda.synchronize(); print("after solve %.1f GB" % used())
g.setup(); torch.cuda.synchronize(); print("after 2nd setup %.1f GB" % used())
print(g.stats()["rows"], g.stats()["nnz"])
