import os, sys
sys.path.insert(0, os.getcwd())
import torch
from paper_1701_01170_b200.generators import rmat_device_graph
from paper_1701_01170_b200.primitives.pagerank import pagerank_device
dg = rmat_device_graph(24, 16, 0)
pagerank_device(dg, 0.85, 0.0, 20)
print(min(pagerank_device(dg, 0.85, 0.0, 20)[1].device_ms for _ in range(2)))
