"""Diagnostics: one DP round at world size 1 with progress prints (scratch)."""
import faulthandler, os, sys, time
faulthandler.dump_traceback_later(90, exit=True)
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import torch.distributed as dist
import workloads
from paper_2304_11745_b200 import gacer as G
from paper_2304_11745_b200.runtime import Session
os.environ.setdefault("MASTER_ADDR", "127.0.0.1"); os.environ.setdefault("MASTER_PORT", "29533")
dist.init_process_group("nccl", rank=0, world_size=1)
warm = torch.ones(4, device="cuda")
dist.all_reduce(warm); torch.cuda.synchronize(); print("nccl warm", flush=True)
g = workloads.build_model("resnet50", 64)
p = workloads.make_params(g, 3, "fp32")
s = Session([(g, p, 4, "bf16", {"train": True})], num_ctas=136, watchdog_ms=5000)
s.set_input(0, workloads.make_input(g, 4, 3, "bf16")); s.set_labels(0, workloads.make_labels(4, 3))
s.run(); torch.cuda.synchronize(); print("plain round ok", flush=True)
G.gacer_train_set_allreduce(0, True)
bks = G.gacer_train_buckets(0, 4 << 20); print("buckets", bks, flush=True)
_, _, grads, _ = s.train_state(0)
stream, comm = torch.cuda.Stream(), torch.cuda.Stream()
for mode in ("gate_only", "wait_only", "full"):
    G.gacer_run_round_async(stream.cuda_stream)
    with torch.cuda.stream(comm):
        if mode != "gate_only":
            for off, n in bks:
                G.gacer_stream_wait_grads(comm.cuda_stream, 0, off, n)
                if mode == "full":
                    dist.all_reduce(grads[off:off + n])
        G.gacer_stream_open_grad_gate(comm.cuda_stream, 0)
    t0 = time.time()
    while not (stream.query() and comm.query()) and time.time() - t0 < 20:
        time.sleep(0.05)
    print(mode, "stream done", stream.query(), "comm done", comm.query(), flush=True)
    if not (stream.query() and comm.query()):
        print(G.gacer_last_error()); break
s.close()
dist.destroy_process_group()
print("ok")
