"""Time the config-5 refine pass (bench.bench_refine) in isolation."""
import argparse, os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
ap = argparse.ArgumentParser()
ap.add_argument("--steps", type=int, default=3)
args = ap.parse_args()
print(json.dumps(bench.bench_refine(torch.device("cuda"), args)))
