"""RMSProp alone on one configs[1] batch's gradients: consume=False (the
bench side measurement) vs consume=True (the training step: the update also
zeroes the gradient rows it read).  CUDA events around the update only."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2307_15333_b200 import scenes  # noqa: E402
from paper_2307_15333_b200.optim import RmsPropState, rmsprop_step  # noqa: E402
from paper_2307_15333_b200.render import BackpropWorkspace, render_and_backprop  # noqa: E402


def main():
    dev = torch.device("cuda")
    tree = scenes.config2_scene(device=dev)
    o, d, t = bench.build_training_pool(tree, dev)
    g = torch.Generator(device=dev)
    g.manual_seed(1)
    idx = torch.randperm(o.shape[0], generator=g, device=dev)[: 1 << 20]
    ws = BackpropWorkspace.for_tree(tree)
    _, grads, _ = render_and_backprop(tree, o, d, t, 1.0, 1e-4, workspace=ws, ray_index=idx)
    saved = (ws.dsigma.clone(), ws.dsh_store.clone())
    sig0, sh0 = tree._sigma.clone(), tree._sh_store.clone()
    state = RmsPropState(tree)
    for consume in (False, True, False, True):
        ts = []
        for rep in range(6):
            ws.dsigma.copy_(saved[0])
            ws.dsh_store.copy_(saved[1])
            tree._sigma.copy_(sig0)
            tree._sh_store.copy_(sh0)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            rmsprop_step(tree, grads, state, consume=consume)
            b.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
        print(f"consume={consume}: {sum(ts[1:]) / 5:.3f} ms")


if __name__ == "__main__":
    main()
