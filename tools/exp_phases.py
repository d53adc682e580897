"""Per-phase device time of the bench training step (events on the main stream)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
from paper_2307_15333_b200 import scenes, _lib
from paper_2307_15333_b200 import render as R
from paper_2307_15333_b200.optim import RmsPropState, StepWorkspace, rmsprop_step
from paper_2307_15333_b200.signals import SignalBuffer
dev = torch.device("cuda")
tree = scenes.config2_scene(device=dev)
o_all, d_all, t_all = bench.build_training_pool(tree, dev)
g = torch.Generator(device=dev); g.manual_seed(7)
perm = torch.randperm(o_all.shape[0], generator=g, device=dev)
st = RmsPropState(tree); buf = SignalBuffer(tree); sws = StepWorkspace(tree, buf); ws = sws.ws
side = torch.cuda.Stream(dev)
N = 1 << 20
plans = {0: R.plan_batch(tree, o_all, d_all, perm[:N], stream=side)}
E = lambda: torch.cuda.Event(enable_timing=True)
acc = {}
for k in range(12):
    idx = perm[k * N:(k + 1) * N]
    plans[k + 1] = R.plan_batch(tree, o_all, d_all, perm[(k + 1) * N:(k + 2) * N], stream=side)
    p = plans.pop(k)
    e = [E() for _ in range(5)]
    e[0].record()
    ws.loss.zero_(); ws.touched.zero_()
    e[1].record()
    ev = [E(), E()]
    loss, grads, _ = R.render_and_backprop(tree, o_all, d_all, t_all, 1.0, 1e-4, grad_scale=2.0 / N, workspace=ws,
                                           accumulate=True, ray_index=idx, plan=p, kernel_events=ev)
    e[2].record()
    rmsprop_step(tree, grads, st, consume=True)
    e[3].record()
    torch.cuda.synchronize()
    if k >= 4:
        for name, a, b in (("memsets", e[0], e[1]), ("bwd call (wait+sched+bwd+update)", e[1], e[2]), ("bwd kernel", ev[0], ev[1]), ("rmsprop", e[2], e[3]), ("total", e[0], e[3])):
            acc.setdefault(name, []).append(a.elapsed_time(b))
for k, v in acc.items():
    print(f"{k:40s} {sum(v) / len(v):.3f} ms")
