"""Compare backward outputs of two kernel-flag settings on the config-2 batch.

    python tools/check_flags.py 0 8192
touched must be identical; gradients / signal / loss agree to fp32-atomic noise."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2307_15333_b200 import scenes  # noqa: E402
from paper_2307_15333_b200.render import BackpropWorkspace, render_and_backprop  # noqa: E402


def run(tree, o, d, t, flags):
    ws = BackpropWorkspace.for_tree(tree)
    loss, g, sig = render_and_backprop(tree, o, d, t, 1.0, 1e-4, workspace=ws, kernel_flags=flags)
    return float(loss), ws.touched.clone(), ws.dsigma.clone(), ws.dsh_store.clone(), sig.clone()


def main():
    fa, fb = int(sys.argv[1]), int(sys.argv[2])
    dev = torch.device("cuda")
    tree = scenes.config2_scene(device=dev)
    o_all, d_all, t_all = bench.build_training_pool(tree, dev)
    g = torch.Generator(device=dev)
    g.manual_seed(7)
    idx = torch.randperm(o_all.shape[0], generator=g, device=dev)[: 1 << 20]
    o, d, t = o_all[idx].contiguous(), d_all[idx].contiguous(), t_all[idx].contiguous()
    A, B = run(tree, o, d, t, fa), run(tree, o, d, t, fb)
    print("loss", A[0], B[0])
    print("touched identical:", bool(torch.equal(A[1], B[1])), int(A[1].sum()), int(B[1].sum()))
    for name, x, y in (("dsigma", A[2], B[2]), ("dsh", A[3], B[3]), ("signal", A[4], B[4])):
        err = (x.double() - y.double()).abs().max().item()
        scale = x.double().abs().max().item()
        print(f"{name}: max abs diff {err:.3e} (max |x| {scale:.3e})")


if __name__ == "__main__":
    main()
