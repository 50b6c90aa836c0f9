"""Per-iteration cost breakdown of the partitioned path at world size 1 (NCCL)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("MASTER_ADDR", "127.0.0.1"); os.environ.setdefault("MASTER_PORT", "29533")
os.environ.setdefault("RANK", "0"); os.environ.setdefault("WORLD_SIZE", "1")
import torch, torch.distributed as dist
import paper_2203_09284_b200 as fb
from paper_2203_09284_b200.dist import B200Part, TorchExchange
torch.cuda.set_device(0)
dist.init_process_group("nccl", device_id=torch.device("cuda", 0))
s = fb.torch_stream_handle()
full = fb.DeviceGraph.generate_uniform(1 << 22, 16, 2, stream=s)
part = B200Part(full, 1, 0, stream=s); full.close()
ex = TorchExchange(); S = part.slice
a = torch.zeros(S, dtype=torch.float64, device="cuda"); b = torch.zeros_like(a); pair = torch.zeros(2, dtype=torch.float64, device="cuda")
part.init(a); torch.cuda.synchronize()
cfg = fb.PageRankConfig(threshold=1e-10)
def t(f, reps=20):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    for _ in range(reps): f()
    torch.cuda.synchronize(); return (time.perf_counter() - t0) / reps * 1e6
print("sweep only      us", t(lambda: part.sweep(fb.ENGINE_EC, cfg, a, b, pair)))
print("allgather slices us", t(lambda: ex.allgather_slices(b, S)))
print("allgather pairs  us", t(lambda: ex.allgather_pairs(pair)))
print("pairs .cpu()     us", t(lambda: ex.allgather_pairs(pair).cpu()))
def it():
    part.sweep(fb.ENGINE_EC, cfg, a, b, pair); ex.allgather_slices(b, S); ex.allgather_pairs(pair).cpu()
print("full iteration   us", t(it))
dist.destroy_process_group()
