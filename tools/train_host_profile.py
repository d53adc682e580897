"""Host (Python) cost of the drop-in training loop at small batches:
cProfile of train_epoch over a ResidentRays dataset, 4096-ray batches."""
import cProfile
import os
import pstats
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2307_15333_b200 import scenes  # noqa: E402
from paper_2307_15333_b200.optim import ResidentRays, RmsPropState, TrainConfig, train_epoch  # noqa: E402
from paper_2307_15333_b200.signals import SignalBuffer  # noqa: E402


class Data:
    def __init__(self, o, d, t):
        self.origins, self.dirs, self.targets, self.heldout = o, d, t, []


def main():
    dev = torch.device("cuda")
    tree = scenes.config2_scene(device=dev)
    o, d, t = bench.build_training_pool(tree, dev)
    sel = torch.randperm(o.shape[0], device=dev)[: 1 << 22]
    data = Data(o[sel].cpu().numpy(), d[sel].cpu().numpy(), t[sel].cpu().numpy())
    cfg = TrainConfig(batch_size=int(os.environ.get("BATCH", "4096")), background=1.0, device_shuffle=True)
    pool = ResidentRays(tree, data, cfg.batch_size)
    state, buf = RmsPropState(tree), SignalBuffer(tree)
    rng = np.random.default_rng(0)
    train_epoch(tree, pool, state, buf, cfg, rng)
    pr = cProfile.Profile()
    pr.enable()
    train_epoch(tree, pool, state, buf, cfg, rng)
    pr.disable()
    pstats.Stats(pr).sort_stats("tottime").print_stats(18)


if __name__ == "__main__":
    main()
