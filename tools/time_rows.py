"""Time the SURVEY 8(f) row kernels (bench.py's next_rows section) standalone."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import argparse
import torch
import bench

args = argparse.Namespace(steps=5)
peaks, _ = bench.measured_peaks()
print(json.dumps(bench.bench_next_rows(args, torch.device("cuda"), peaks), indent=1))
