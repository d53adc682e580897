"""PeerExchange end to end under torchrun (N >= 1): a few train_steps with the
fused peer update vs the same steps with the plain update, on every rank."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", "0")))
    dist.init_process_group("nccl", device_id=torch.device("cuda", torch.cuda.current_device()))
    from helpers import irregular_tree, ray_batch
    from paper_2307_15333_b200.optim import RmsPropState, StepWorkspace, train_step
    from paper_2307_15333_b200.parallel import PeerExchange, shard_bounds
    from paper_2307_15333_b200.signals import SignalBuffer
    from paper_2307_15333_b200.scene_io import load_tree_bytes, tree_bytes
    base = irregular_tree(3, 16, depth=3, splits=40, max_depth=6, device="cuda")
    blob = tree_bytes(base)
    o, d = ray_batch(4, 1 << 16)
    t = np.random.default_rng(5).uniform(0, 1, (o.shape[0], 3))
    o, d, t = (torch.from_numpy(x).cuda() for x in (o, d, t))
    n = o.shape[0]
    lo, hi = shard_bounds(n, rank, world)
    gs = 2.0 / n
    trees = []
    for mode in ("peer", "plain"):
        tree = load_tree_bytes(blob, device="cuda")
        st = RmsPropState(tree)
        buf = SignalBuffer(tree)
        sws = StepWorkspace(tree, buf)
        ex = PeerExchange(tree, st, sws) if mode == "peer" else None
        for k in range(3):
            if mode == "peer":
                train_step(tree, o[lo:hi], d[lo:hi], t[lo:hi], st, buf, sws, 0.5, grad_scale=gs, exchange=ex)
            else:  # plain: every rank processes the whole batch
                train_step(tree, o, d, t, st, buf, sws, 0.5, grad_scale=gs)
        torch.cuda.synchronize()
        trees.append(tree)
    a, b = trees
    ds = (a.sigma - b.sigma).abs().max().item()
    dh = (a.sh - b.sh).abs().max().item()
    print(f"rank {rank}/{world}: max |dsigma| {ds:.3e} max |dsh| {dh:.3e}", flush=True)
    ok = ds < 1e-4 and dh < 1e-4
    print("PEER_OK" if ok else "PEER_MISMATCH", flush=True)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
