"""Stage step on the cfg3 shape (1M x 1000 f32 logits) a few times, for ncu."""
import sys
import torch
sys.path.insert(0, ".")
from paper_2406_14424_b200.stage import stage_step
x = torch.randn((1_000_000, 1000), device="cuda")
for kind in ("margin", "entropy", "margin", "entropy"):
    r = stage_step(x, 0.05, kind=kind)
torch.cuda.synchronize()
print("done")
