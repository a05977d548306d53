timeout 300 python scratch/graph_probe.py 2>&1 | tail -6
