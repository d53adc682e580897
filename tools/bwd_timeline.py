"""Wave structure of one backward launch (diagnostic build with per-block
%globaltimer stamps: python tools/build_variants.py diag=DOT_DIAG_FLAGS, then
DOT_LIB_PATH=tools/variants/lib_diag.so python tools/bwd_timeline.py)."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2307_15333_b200 import _lib, scenes  # noqa: E402
from paper_2307_15333_b200.render import BackpropWorkspace, render_and_backprop  # noqa: E402


def main():
    dev = torch.device("cuda")
    tree = scenes.config2_scene(device=dev)
    o, d, t = bench.build_training_pool(tree, dev)
    g = torch.Generator(device=dev)
    for k in range(4):  # warm the schedule on different batches, then time a fresh one
        g.manual_seed(100 + k)
        idx = torch.randperm(o.shape[0], generator=g, device=dev)[: 1 << 20]
        ws = BackpropWorkspace.for_tree(tree)
        render_and_backprop(tree, o, d, t, 1.0, ray_index=idx, workspace=ws)
    torch.cuda.synchronize()
    nb = (1 << 20) // 32
    buf = np.zeros(2 * nb, dtype=np.uint64)
    _lib.load().dot_diag_timeline(buf.ctypes.data_as(ctypes.c_void_p), ctypes.c_int(nb))
    t0, t1 = buf[0::2].astype(np.float64), buf[1::2].astype(np.float64)
    base = t0.min()
    t0, t1 = (t0 - base) / 1e3, (t1 - base) / 1e3  # us
    span = t1.max()
    dur = t1 - t0
    print(f"kernel span {span:.0f} us, warp duration p50 {np.median(dur):.0f} p99 {np.percentile(dur, 99):.0f} "
          f"max {dur.max():.0f} us, last warp start {t0.max():.0f} us ({100 * t0.max() / span:.0f} %)")
    grid = np.linspace(0, span, 101)
    active = np.array([np.sum((t0 <= x) & (t1 > x)) for x in grid])
    peak = active.max()
    print("active warps over the kernel (every 10 %):", [int(a) for a in active[::10]])
    low = grid[active < 0.5 * peak]
    print(f"time with < 50 % of peak warps active: {100 * (active < 0.5 * peak).mean():.0f} % of the span")
    late = np.argsort(t1)[-15:]
    print("latest-ending warps (launch pos, start us, duration us):",
          [(int(i), int(t0[i]), int(dur[i])) for i in late])
    longw = dur > 400
    print(f"warps > 400 us: {int(longw.sum())}; their start times p50 {np.median(t0[longw]):.0f} "
          f"p90 {np.percentile(t0[longw], 90):.0f} max {t0[longw].max():.0f} us; launch positions p90 "
          f"{np.percentile(np.nonzero(longw)[0], 90):.0f} of {nb}")
    # what a perfect packing of the same warp durations would take
    print(f"sum of warp durations / (peak concurrency) = {dur.sum() / peak:.0f} us (vs span {span:.0f})")


if __name__ == "__main__":
    main()
