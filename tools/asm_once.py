import sys; sys.path.insert(0, "/root/repo")
import torch, synth
from paper_1812_05540_b200 import assemble
fl = synth.fields("C5", x_rand=False)
d = {k: torch.from_numpy(fl[k]).cuda() for k in ("E", "perm", "phi", "sat", "pres", "well")}
for _ in range(2):
    ap = assemble(fl["params"], d); torch.cuda.synchronize(); del ap
