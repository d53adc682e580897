"""How fair is the C oracle port as a stand-in for the reference's speed?

Runs in the BUILD container only (needs /root/reference): times the
reference's own public `octrf.render.render_and_backprop` (Numba, all host
threads, JIT warmed up) and the C oracle port (`oracle/dot_oracle.c`, OpenMP,
same thread count) on the same configs[1] scene (written with our save_tree,
loaded with octrf.load_tree: byte-compatible .dot1) and the same ray sample;
checks that both return the same loss.  Prints one line per implementation.

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba_cache \
        python tools/calibrate_port.py [--rays 65536]
"""
import argparse
import os
import sys
import tempfile
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import bench  # noqa: E402
from oracle import oracle as O  # noqa: E402
from paper_2307_15333_b200 import scenes  # noqa: E402
from paper_2307_15333_b200.scene_io import save_tree  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rays", type=int, default=1 << 16)
    ap.add_argument("--reps", type=int, default=3)
    args = ap.parse_args()
    import octrf.render as R
    from octrf.scene_io import load_tree
    tree = scenes.config2_scene(device="cpu")
    tree._host()
    with tempfile.TemporaryDirectory() as tmp:
        path = os.path.join(tmp, "c2.dot1")
        save_tree(tree, path)
        ref_tree = load_tree(path)
    focal, poses = scenes.hemisphere_cameras(100, bench.W, bench.H, bench.RADIUS, seed=3)
    rng = np.random.default_rng(0)
    o, d = bench.view_rays_np(focal, poses[0]) if hasattr(bench, "view_rays_np") else (None, None)
    if o is None:
        import torch
        ot, dt = bench.view_rays_torch(focal, poses[0], torch.device("cpu"))
        o, d = ot.numpy(), dt.numpy()
    pick = rng.choice(o.shape[0], args.rays, replace=False)
    o, d = np.ascontiguousarray(o[pick]), np.ascontiguousarray(d[pick])
    tgt = rng.uniform(0.0, 1.0, (args.rays, 3))
    threads = O.num_threads()
    R.render_and_backprop(ref_tree, o[:1024], d[:1024], tgt[:1024], bench.BG, bench.EPS)  # JIT
    for name, fn in (("reference octrf (Numba)", lambda: R.render_and_backprop(ref_tree, o, d, tgt, bench.BG, bench.EPS)),
                     ("C oracle port (OpenMP)", lambda: O.render_and_backprop(tree, o, d, tgt, bench.BG, bench.EPS))):
        best, loss = 1e9, None
        for _ in range(args.reps):
            t0 = time.perf_counter()
            out = fn()
            best = min(best, time.perf_counter() - t0)
            loss = float(out[0])
        print(f"{name}: {args.rays / best:.3e} rays/s ({best:.2f} s for {args.rays} rays, "
              f"{threads} threads), loss {loss:.12g}", flush=True)


if __name__ == "__main__":
    main()
