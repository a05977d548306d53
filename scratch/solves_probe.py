import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
import paper_2409_20027_b200 as P
print(json.dumps(bench.single_solve_leg(torch, P, cpu=True)))
