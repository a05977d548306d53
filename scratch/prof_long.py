"""Profile driver: config-4 time-sharded LQR solve at world 1 (one solve after warm-up)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
steps = int(sys.argv[1]) if len(sys.argv) > 1 else 1
c0 = int(sys.argv[2]) if len(sys.argv) > 2 else 0
c1 = int(sys.argv[3]) if len(sys.argv) > 3 else 0
print(c0, c1, bench.long_horizon_leg(torch, 1, 0, steps=steps, chunk0=c0, chunk=c1))
