"""Leaf counts of the config-4 scene for a few split thresholds."""
import sys, time
sys.path.insert(0, ".")
import torch
from paper_2307_15333_b200 import scenes
for thr in [float(x) for x in sys.argv[1:]] or [300.0, 400.0, 600.0]:
    torch.cuda.synchronize(); t = time.time()
    try:
        tr = scenes.config4_scene(device="cuda", split_thr=thr)
    except torch.OutOfMemoryError:
        print(thr, "OOM"); torch.cuda.empty_cache(); continue
    torch.cuda.synchronize()
    print(thr, "leaves", tr.leaf_count, "nodes", tr.capacity, "s", round(time.time() - t, 2),
          "levels", list(tr.topology().level_offsets), flush=True)
    del tr; torch.cuda.empty_cache()
