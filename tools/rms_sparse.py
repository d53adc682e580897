"""RMSProp dense (capacity-sized grid) vs sparse (touched-row list) on the
configs[1] tree for batches of 2^12 .. 2^20 rays: one backward fills the
gradients / touched mask, then each update is timed alone (consume=False)."""
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
    state = RmsPropState(tree)
    g = torch.Generator(device=dev)
    g.manual_seed(1)
    for lg in (12, 14, 16, 17, 18, 19, 20):
        idx = torch.randperm(o.shape[0], generator=g, device=dev)[: 1 << lg]
        ws = BackpropWorkspace.for_tree(tree)
        _, grads, _ = render_and_backprop(tree, o, d, t, 1.0, 1e-4, workspace=ws, ray_index=idx)
        touched = int(ws.touched.sum())
        res = []
        for sparse in (False, True):
            for _ in range(2):
                rmsprop_step(tree, grads, state, sparse=sparse)
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            for _ in range(5):
                rmsprop_step(tree, grads, state, sparse=sparse)
            b.record()
            torch.cuda.synchronize()
            res.append(a.elapsed_time(b) / 5)
        print(f"2^{lg} rays: touched {touched:8d} ({touched / tree.capacity:.3f} of capacity)  "
              f"dense {res[0]:.3f} ms  sparse {res[1]:.3f} ms")


if __name__ == "__main__":
    main()
