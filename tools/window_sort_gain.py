"""What grouping rays of similar cost into the same warp could buy: for the
plan's key-ordered 2^20-ray batch, the sum over warps of the warp's max
per-ray cost (composited + post-cut / 2 -- the backward's lane-serial work)
when rays are re-sorted by cost inside windows of G consecutive rays (G = 32:
today's order)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2307_15333_b200 import scenes  # noqa: E402
from paper_2307_15333_b200.render import PoolRank, plan_batch, pool_rank, ray_costs  # noqa: E402


def main():
    dev = torch.device("cuda")
    tree = scenes.config2_scene(device=dev)
    o, d, t = bench.build_training_pool(tree, dev)
    pr = pool_rank(tree, o, d)
    costs = ray_costs(tree, o, d)
    o, d, costs = pr.permute(o, d, costs)
    g = torch.Generator(device=dev)
    g.manual_seed(3)
    idx = torch.randperm(o.shape[0], generator=g, device=dev)[: 1 << 20]
    p = plan_batch(tree, o, d, idx, rank=PoolRank.identity(o.shape[0], dev))
    c = costs[p.idx].float()
    n = c.shape[0]
    base = c.view(-1, 32).amax(1).sum().item()
    print(f"sum of per-ray cost {c.sum().item():.4g}; key order: sum of warp max {base:.4g} "
          f"(lane efficiency {c.sum().item() / (32 * base):.3f})")
    for G in (64, 128, 256, 512, 1024, 4096):
        cs = c.view(-1, G).sort(dim=1, descending=True).values.reshape(n)
        s = cs.view(-1, 32).amax(1).sum().item()
        print(f"window {G:5d}: sum of warp max {s:.4g} ({s / base:.3f} of key order; lane eff "
              f"{c.sum().item() / (32 * s):.3f})")


if __name__ == "__main__":
    main()
