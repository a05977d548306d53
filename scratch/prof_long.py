"""Profile driver: config-4 time-sharded LQR solve at world 1 (one solve after warm-up)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
print(bench.long_horizon_leg(torch, 1, 0, steps=int(sys.argv[1]) if len(sys.argv) > 1 else 1))
