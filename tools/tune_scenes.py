"""Print leaf counts / build times of the adaptive scenes (used to pick thresholds)."""
import sys, time
sys.path.insert(0, ".")
import torch
from paper_2307_15333_b200 import scenes
for seed, depth, thr in [(2, 9, 800.0), (5, 10, 250.0), (5, 10, 400.0), (5, 10, 600.0)]:
    torch.cuda.synchronize(); t = time.time()
    tr = scenes.adaptive_tree(scenes.BlobField.make(seed=seed, n_blobs=64), max_depth=depth,
                              basis_count=16, split_thr=thr, min_depth=4, device="cuda")
    torch.cuda.synchronize()
    print(seed, depth, thr, "leaves", tr.leaf_count, "nodes", tr.capacity, "s", round(time.time() - t, 2),
          "levels", list(tr.topology().level_offsets), flush=True)
    del tr; torch.cuda.empty_cache()
