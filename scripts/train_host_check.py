"""Host issue time vs device time of the sequential training step (ResNet-50,
B=64, 224^2): how close the Python-sequenced step is to being host-bound."""
import sys, time, numpy as np, torch
sys.path.insert(0, "/root/repo")
import workloads
from paper_2304_11745_b200 import gacer as G
from paper_2304_11745_b200.train_driver import SequentialTrainer
g = workloads.build_model("resnet50", 224); B = 64
params = workloads.make_params(g, 7, "fp32"); x = workloads.make_input(g, B, 7, "bf16"); labels = workloads.make_labels(B, 7)
G.gacer_init(0)
tr = SequentialTrainer(g, params, B)
xp = np.zeros((B, 224, 224, 8), np.float32); xp[..., :3] = x.transpose(0, 2, 3, 1)
xd = torch.from_numpy(xp).to(torch.bfloat16).cuda(); lab = torch.from_numpy(labels).cuda()
for _ in range(3): tr.step(xd, lab)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
t0 = time.perf_counter(); e0.record()
for _ in range(5): tr.step(xd, lab)
t1 = time.perf_counter(); e1.record(); e1.synchronize(); t2 = time.perf_counter()
print("issue ms/step", (t1 - t0) / 5 * 1e3, "gpu ms/step", e0.elapsed_time(e1) / 5, "wall ms/step", (t2 - t0) / 5 * 1e3)
G.gacer_shutdown()
