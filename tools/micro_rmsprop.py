"""Time rmsprop_step on the config-2 scene (all rows touched)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2307_15333_b200 import scenes
from paper_2307_15333_b200.optim import RmsPropState, rmsprop_step
from paper_2307_15333_b200.render import BackpropWorkspace, GradBuffer
tree = scenes.config2_scene(device="cuda")
ws = BackpropWorkspace.for_tree(tree)
ws.dsigma.normal_(); ws.dsh_store.normal_(); ws.touched.fill_(1)
st = RmsPropState(tree)
g = GradBuffer(ws.dsigma, ws.dsh_store[:, :48], ws.touched, tree.generation, ws.dsh_store)
for _ in range(3):
    rmsprop_step(tree, g, st)
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(10):
    rmsprop_step(tree, g, st)
b.record(); torch.cuda.synchronize()
ms = a.elapsed_time(b) / 10
rows = tree.capacity
byts = rows * (1 + 4 + 8 + 4 + 192 + 384 + 192) + rows * (4 + 8 + 192 + 384)
print(f"rmsprop {ms:.3f} ms  {byts / ms / 1e6:.0f} GB/s ({rows} rows)")
