import faulthandler, socket, sys
sys.path.insert(0, '/root/repo')
faulthandler.dump_traceback_later(90, exit=True)
import torch, torch.distributed as dist
from paper_2605_11537_b200.engine import MoEPipeline, PipelineConfig
with socket.socket() as so:
    so.bind(("127.0.0.1", 0)); port = so.getsockname()[1]
dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1, device_id=torch.device("cuda", 0))
cfg = PipelineConfig(num_layers=3, num_experts=32, d_model=256, d_ff=512, tokens=4096, sru_layers=3, capacity=64, seed=5)
s = torch.cuda.Stream()
with torch.cuda.stream(s):
    b = MoEPipeline(cfg)
    emb, _, _ = b.wl.batch(cfg.tokens)
    b.enable_expert_parallel(peer_cap=None)
    b.force_collectives = True
    xb = emb.clone()
    print("eager step", flush=True)
    b.step(xb); torch.cuda.synchronize()
    print("capture", flush=True)
    g = b.capture(xb)
    print("captured; replay", flush=True)
    g.replay(); torch.cuda.synchronize()
    print("replayed", flush=True)
    g.destroy(); torch.cuda.synchronize()
print("destroying pg", flush=True)
dist.destroy_process_group()
