"""One training GEMM launch for an ncu capture: conv dgrad (or wgrad) of a
ResNet-50 layer1 3x3 conv at B=64 (56x56, 64 -> 64 channels).

usage: python scripts/one_train_gemm.py [dgrad|wgrad]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2304_11745_b200 import gacer as G  # noqa: E402

which = sys.argv[1] if len(sys.argv) > 1 else "dgrad"
B, H, C, K = 64, 56, 64, 3
G.gacer_init(0)
x = torch.randn(B, H, H, C, device="cuda").to(torch.bfloat16)
dy = torch.randn(B, H, H, C, device="cuda").to(torch.bfloat16)
w = torch.randn(C, C, K, K, device="cuda") * 0.05
out = torch.empty_like(x) if which == "dgrad" else torch.empty_like(w)
fn = G.conv_dgrad_workspace if which == "dgrad" else G.conv_wgrad_workspace
nb = fn(B, H, H, C, C, K, K, 1, 1, 1)
ws = torch.empty(nb + 256, dtype=torch.uint8, device="cuda")
base = (ws.data_ptr() + 255) // 256 * 256
for _ in range(3):
    if which == "dgrad":
        G.conv_dgrad(dy.data_ptr(), w.data_ptr(), B, H, H, C, C, K, K, 1, 1, 1, out.data_ptr(), base, nb)
    else:
        G.conv_wgrad(x.data_ptr(), dy.data_ptr(), B, H, H, C, C, K, K, 1, 1, 1, out.data_ptr(), base, nb)
torch.cuda.synchronize()
G.gacer_shutdown()
print("ok", which)
