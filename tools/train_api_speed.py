"""The drop-in training loop's speed: optim.train_epoch over a ResidentRays
dataset (configs[1] scene, 2^23 rays of the training views, 2^20-ray
batches) -- per-batch time of whole epochs, against bench.py's step."""
import os
import sys
import time

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
    g = torch.Generator(device=dev)
    g.manual_seed(2)
    sel = torch.randperm(o.shape[0], generator=g, device=dev)[: 1 << 23]
    data = Data(o[sel].cpu().numpy(), d[sel].cpu().numpy(), t[sel].cpu().numpy())
    del o, d, t
    torch.cuda.empty_cache()
    bs = int(os.environ.get("BATCH", str(1 << 20)))
    cfg = TrainConfig(batch_size=bs, background=1.0, device_shuffle=os.environ.get("DEVICE_SHUFFLE") == "1")
    print("device_shuffle", cfg.device_shuffle)
    c0 = time.perf_counter()
    pool = ResidentRays(tree, data, cfg.batch_size, cfg.early_stop_eps)
    torch.cuda.synchronize()
    print(f"ResidentRays setup {time.perf_counter() - c0:.2f} s (upload, rank, costs)")
    state, buf = RmsPropState(tree), SignalBuffer(tree)
    rng = np.random.default_rng(0)
    train_epoch(tree, pool, state, buf, cfg, rng)  # warm-up epoch
    for ep in range(3):
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        loss = train_epoch(tree, pool, state, buf, cfg, rng)
        b.record()
        torch.cuda.synchronize()
        ms = a.elapsed_time(b)
        nb = ((1 << 23) + bs - 1) // bs
        print(f"epoch of {nb} batches: {ms:.2f} ms = {ms / nb:.3f} ms per {bs}-ray batch "
              f"({(1 << 23) / (ms / 1e3):.3e} rays/s), loss {loss:.5f}")


if __name__ == "__main__":
    main()
