import cProfile, pstats, sys, time
sys.path.insert(0, '/root/repo')
import numpy as np, torch
from paper_2605_11537_b200.engine import MoEPipeline, PipelineConfig
from paper_2605_11537_b200.placement import DeviceState, apply_batch, execution_map
from paper_2605_11537_b200.planner import plan_layers_with_fallback
from paper_2605_11537_b200.predictor import predict_batch
from paper_2605_11537_b200.router_oracle import moe_forward
from paper_2605_11537_b200.workload import Batch
with torch.cuda.stream(torch.cuda.Stream()):
    pipe = MoEPipeline(PipelineConfig())
    b = [pipe.wl.batch(16384) for _ in range(2)]
    params, sru = pipe.toy_params(), pipe.sru_params()
    host = [Batch(k, x[0].cpu().numpy(), x[2].cpu().numpy().astype(np.int64)) for k, x in enumerate(b)]
    state = DeviceState(12, 296)
    def one(batch):
        t0 = time.perf_counter(); table = predict_batch(batch, sru); t1 = time.perf_counter()
        plan = plan_layers_with_fallback(table, 296); t2 = time.perf_counter()
        apply_batch(state, table, plan); t3 = time.perf_counter()
        _, ex, _ = execution_map(state, batch.oracle_routing); t4 = time.perf_counter()
        out = moe_forward(batch.embeddings, params, ex); t5 = time.perf_counter()
        return [t1-t0, t2-t1, t3-t2, t4-t3, t5-t4]
    one(host[0]); one(host[1])
    for k in range(3):
        print(["%.1f ms" % (v*1e3) for v in one(host[k % 2])])
    pr = cProfile.Profile(); pr.enable(); one(host[0]); pr.disable()
    pstats.Stats(pr).sort_stats("tottime").print_stats(18)

    # moe_forward phases
    import paper_2605_11537_b200.router_oracle as R
    dev = torch.device("cuda")
    dm = R._device_moe(params, dev)
    batch = host[0]
    _, ex, _ = execution_map(state, batch.oracle_routing)
    for _ in range(2):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        x = R._stream_device(batch.embeddings, 768, dm.dp, dev); torch.cuda.synchronize(); t1 = time.perf_counter()
        pl = R._validated_placement(ex, params, 16384, dev); torch.cuda.synchronize(); t2 = time.perf_counter()
        R._run_layers_device(x, dm, placement=pl); torch.cuda.synchronize(); t3 = time.perf_counter()
        out = x[:, :768].cpu().numpy(); t4 = time.perf_counter()
        print("moe_forward phases: upload %.1f  placement %.1f  layers %.1f  download %.1f ms" % ((t1-t0)*1e3, (t2-t1)*1e3, (t3-t2)*1e3, (t4-t3)*1e3))
