import sys, time, torch
sys.path.insert(0, '.')
import bench
class A: source=0; edge_factor=16; scale=24
print(bench.scale27(A(), 6547.0))
