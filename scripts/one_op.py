"""Run one conv op (conv+BN+ReLU) tenant in executor mode a few rounds (for ncu)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, workloads
from paper_2304_11745_b200.runtime import Session
cin, cout, k, st, pad, hw, B = [int(v) for v in sys.argv[1:8]]
g = workloads.Graph("op", cin, hw, hw)
g.relu(g.bn(g.conv(0, cin, cout, k, st, pad), cout))
s = Session([(g, workloads.make_params(g, 1), B, "bf16")])
s.set_input(0, workloads.make_input(g, B, 1))
for _ in range(4):
    s.run()
torch.cuda.synchronize()
s.close()
