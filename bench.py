#!/usr/bin/env python
"""Benchmark: Switch-base-128 MoE-MPMC inference (BASELINE.json config 3) on B200.

One step = one batch of T tokens through the whole hot path on the GPU:
SRU predictor (10 layers) -> load histogram -> capped replica plan -> residency
/ token walk -> 12 x [top-1 router -> execution map over replicas -> gather ->
grouped expert GEMM1 (ReLU) -> grouped GEMM2 + scatter residual combine].

  python bench.py [--gpus N --steps K --warmup W] [--replication on|off|split]
  python bench.py --impl reference ...      # CPU oracle port on the host cores

Prints ONE JSON line (rank 0). Under torchrun (N > 1) every rank runs its own
replica of the pipeline on its own batch (weak scaling, no data-path
collective yet), timed on the device and reduced with MAX over ranks.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "Switch-base-128 MoE tokens/s at 1/2/4/8 B200; grouped-GEMM tensor-pipe %"


def parse_args():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=50)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", choices=["ours", "reference"], default="ours")
    p.add_argument("--replication", choices=["on", "off", "split"], default="on")
    p.add_argument("--tokens", type=int, default=16384)
    p.add_argument("--layers", type=int, default=12)
    p.add_argument("--experts", type=int, default=128)
    p.add_argument("--capacity", type=int, default=296)
    p.add_argument("--demand-unit", type=int, default=128)
    p.add_argument("--predictor", choices=["constructed", "random"], default="constructed")
    p.add_argument("--batches", type=int, default=4, help="distinct synthetic batches cycled over the steps")
    p.add_argument("--cpu-sample-tokens", type=int, default=2048)
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--seed", type=int, default=0)
    p.add_argument("--skew", type=float, default=1.2, help="Zipf skew of the synthetic routing")
    p.add_argument("--no-graph", action="store_true", help="launch kernels one by one instead of a CUDA graph")
    p.add_argument("--l2-persist", type=float, default=1.0, help="persisting-L2 hit ratio for the residual stream")
    p.add_argument("--ffn", choices=["auto", "two", "mt", "fused", "pair"], default="auto")
    p.add_argument("--ep", action="store_true", help="expert-parallel path even at N=1 (always on for N>1)")
    p.add_argument("--ffn-sms", type=int, default=0, help="--overlap on: persistent grid of the expert GEMMs")
    p.add_argument("--pred-sms", type=int, default=0, help="--overlap on: persistent grid of the predictor GEMMs")
    p.add_argument("--overlap", choices=["on", "off"], default="off",
                   help="predictor of batch i+1 on its own stream during batch i (two-actor pipeline)")
    return p.parse_args()


def load_peaks():
    try:
        return json.loads((ROOT / "MEASURED_PEAKS.json").read_text()), "measured"
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}, "fallback"


class ClockSampler:
    """nvidia-smi sampling of SM clocks and throttle reasons during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self.proc = None
        self.nvml = None
        self.stop_evt = threading.Event()
        self.t0 = self.t1 = None

    def mark(self, begin: bool):
        """Bracket the timed region (NVML samples outside it are dropped)."""
        if begin:
            self.t0 = time.time()
        else:
            self.t1 = time.time()

    def _nvml_handle(self):
        """NVML handle of the CUDA device (matched by PCI bus id, so CUDA_VISIBLE_DEVICES cannot mislead it)."""
        import pynvml
        import torch
        pynvml.nvmlInit()
        pr = torch.cuda.get_device_properties(self.index)
        try:
            bus = f"{pr.pci_domain_id:08x}:{pr.pci_bus_id:02x}:{pr.pci_device_id:02x}.0"
            return pynvml, pynvml.nvmlDeviceGetHandleByPciBusId(bus)
        except Exception:
            return pynvml, pynvml.nvmlDeviceGetHandleByIndex(self.index)

    def _nvml_loop(self):
        nv, h = self.nvml
        reasons = nv.nvmlDeviceGetCurrentClocksEventReasons if hasattr(nv, "nvmlDeviceGetCurrentClocksEventReasons") \
            else nv.nvmlDeviceGetCurrentClocksThrottleReasons
        bits = [0x8, 0x40, 0x20, 0x4]  # hw_slowdown, hw_thermal_slowdown, sw_thermal_slowdown, sw_power_cap
        mx = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
        while not self.stop_evt.is_set():
            try:
                sm = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
                r = reasons(h)
                row = [str(sm), str(mx), "0"] + ["Active" if r & b else "Not Active" for b in bits]
                if self.t0 is not None and self.t1 is None:  # inside the timed region only
                    self.rows.append(row)
            except Exception:
                pass
            time.sleep(0.005)

    def start(self):
        try:  # NVML: a sample every ~5 ms (nvidia-smi -lms cannot sample a sub-second timed region)
            self.nvml = self._nvml_handle()
            threading.Thread(target=self._nvml_loop, daemon=True).start()
            return
        except Exception:
            self.nvml = None
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
            return
        threading.Thread(target=self._read, daemon=True).start()

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([c.strip() for c in line.split(",")])

    def stop(self):
        self.stop_evt.set()
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
        time.sleep(0.05)
        sm = [float(r[0]) for r in self.rows if len(r) >= 7 and r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if len(r) >= 7 and r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows if len(r) >= 7 for i in range(4) if r[3 + i] == "Active"})
        loaded = [s for s in sm if s > 0.5 * max(mx or [1])] or sm
        med = sorted(loaded)[len(loaded) // 2] if loaded else None
        return {"sm_mhz": med, "sm_max_mhz": max(mx) if mx else None, "reasons": reasons, "samples": len(self.rows),
                "source": "nvml" if self.nvml is not None else "nvidia-smi"}


def dist_setup():
    import torch

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch.distributed as dist

        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    return world, rank, local


def max_over_ranks(value: float, world: int) -> float:
    if world == 1:
        return value
    import torch
    import torch.distributed as dist

    t = torch.tensor([value], device="cuda", dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def barrier(world: int):
    if world > 1:
        import torch.distributed as dist

        dist.barrier()


def cpu_baseline(args, steps: int = 1, warmup: int = 0):
    from oracle.cpu_pipeline import CpuSample, host_threads

    s = CpuSample(tokens=args.cpu_sample_tokens, L=args.layers, E=args.experts, capacity=args.capacity,
                  demand_unit=args.demand_unit, seed=args.seed, constructed_predictor=args.predictor == "constructed")
    for _ in range(warmup):
        s.run()
    times, br = [], None
    for _ in range(steps):
        t, br = s.run()
        times.append(t)
    total = sum(times)
    return {
        "value": args.cpu_sample_tokens * steps / total,
        "unit": "tokens/s",
        "cores": host_threads(),
        "kind": "port",
        "sample": (f"{args.cpu_sample_tokens} tokens of the config-3 workload through the full chain: float64 SRU "
                   f"predictor ({10} layers), plan/place x{args.layers}, {args.layers} MoE layers (route + exec map + "
                   f"fp32 expert FFN, one layer's expert weights shared by all layers to bound host RAM); "
                   f"numpy/OpenBLAS on all host threads"),
        "ms_per_sample": 1e3 * total / steps,
        "breakdown_s": br,
    }


def run_reference(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    cb = cpu_baseline(args, steps=args.steps, warmup=args.warmup)
    out = {
        "impl": "reference",
        "metric": METRIC,
        "value": cb["value"],
        "unit": "tokens/s",
        "n_gpus": args.gpus,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": cb["ms_per_sample"],
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "f64 predictor / f32 FFN",
        "data": "synthetic",
        "config": config_dict(args, world),
        "cpu_baseline": {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample")},
        "e2e": {"value": cb["value"], "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(out))
    return 0


def config_dict(args, world):
    return {
        "workload": "Switch-base-128 12-layer MoE forward + SRU predictor + replica plan (BASELINE config 3)",
        "model": f"switch-base-{args.experts}",
        "num_layers": args.layers, "num_experts": args.experts, "d_model": 768, "d_ff": 3072,
        "tokens_per_gpu": args.tokens, "global_batch": args.tokens * world, "sru_layers": 10,
        "capacity": args.capacity, "demand_unit": args.demand_unit, "replication": args.replication,
        "predictor": args.predictor, "zipf_skew": args.skew, "parallelism": f"ep{world}" if world > 1 else ("ep1" if args.ep else "single"),
        "l2": "inputs larger than L2 (14.5 GB of expert weights streamed per step)",
    }


def run_ours(args):
    import torch

    world, rank, local = dist_setup()
    from paper_2605_11537_b200.engine import MoEPipeline, PipelineConfig

    cfg = PipelineConfig(num_layers=args.layers, num_experts=args.experts, tokens=args.tokens,
                         capacity=args.capacity, demand_unit=args.demand_unit, replication=args.replication,
                         predictor=args.predictor, ffn=args.ffn, seed=args.seed + rank, skew=args.skew)
    pipe = MoEPipeline(cfg)
    T, d, L = cfg.tokens, cfg.d_model, cfg.num_layers
    ep = world > 1 or args.ep
    if ep:
        pipe.enable_expert_parallel()
    batches = [pipe.wl.batch(T) for _ in range(max(1, args.batches))]
    x = torch.empty(T, d, device="cuda")

    def step(k, events=None):
        emb = batches[k % len(batches)][0]
        x.copy_(emb)
        return pipe.step(x, events)

    if args.l2_persist > 0:
        from paper_2605_11537_b200 import _lib as mplib
        from paper_2605_11537_b200._dev import stream_ptr

        mplib.call("mp_l2_persist", x.data_ptr(), x.numel() * 4, float(args.l2_persist), stream_ptr())
    for k in range(args.warmup):
        step(k)
    torch.cuda.synchronize()

    from paper_2605_11537_b200.engine import DeviceEvent

    ev = [[DeviceEvent() for _ in range(3)] for _ in range(L)]
    graph = None
    overlap = None
    if args.overlap == "on" and not ep and not args.no_graph:
        from paper_2605_11537_b200.engine import OverlappedPipeline

        overlap = OverlappedPipeline(pipe, ev, args.ffn_sms, args.pred_sms)
        overlap.run([b[0] for b in batches], 2)
        torch.cuda.synchronize()
    elif not args.no_graph and not ep:
        # one CUDA graph per step for the timed loop; a second capture with events around every
        # GEMM (event nodes cost ~8 us each inside a graph) is replayed once afterwards for the
        # roofline's per-launch durations
        graph = pipe.capture(x)
        graph_ev = pipe.capture(x, ev)
        for k in range(2):
            x.copy_(batches[k % len(batches)][0])
            graph.replay()
        torch.cuda.synchronize()
    barrier(world)

    clocks = ClockSampler(torch.cuda.current_device() if world == 1 else local)
    clocks.start()
    time.sleep(0.3)
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    barrier(world)
    launches = 0
    clocks.mark(True)
    if overlap is not None:
        overlap.run([b[0] for b in batches], args.steps, timer=(start, end))
        launches = args.steps * overlap.launches  # this repo's kernels only
    else:
        start.record()
        for k in range(args.steps):
            if graph is not None:
                x.copy_(batches[k % len(batches)][0])
                graph.replay()
                launches += graph.launches  # kernel nodes of the step graph (the copy is a memcpy)
            else:
                launches += step(k, ev)
        end.record()
    torch.cuda.synchronize()
    clocks.mark(False)
    elapsed_ms = start.elapsed_time(end)
    clk = clocks.stop()
    elapsed_ms = max_over_ranks(elapsed_ms, world)
    if graph is not None:  # GEMM launch durations: instrumented replays of the same step
        for k in range(3):
            x.copy_(batches[(args.steps - 3 + k) % len(batches)][0])
            graph_ev.replay()
        torch.cuda.synchronize()
    # GEMM launch durations of the last timed step (events recorded inside the step / graph)
    up = [ev[l][0].elapsed_ms(ev[l][1]) for l in range(L)]
    down = [ev[l][1].elapsed_ms(ev[l][2]) for l in range(L)]

    # correctness spot checks on the last step (not timed)
    last = batches[(args.steps - 1) % len(batches)]
    routing_exact = bool((pipe.route.long() == last[2]).all().item()) if not ep else \
        bool((pipe.ep.last_route.long() == last[2][-1]).all().item())
    last_assign = overlap.assign[(args.steps - 1) % 2] if overlap is not None else pipe.assign
    pred_acc = float((last_assign.long() == last[2]).float().mean().item())

    t_up, t_down = sum(up) / len(up), sum(down) / len(down)
    touched = pipe.touched_experts().float().mean().item()
    w_bytes = touched * pipe.expert_weight_bytes()
    # algorithmic bytes of one MoE layer's FFN: every touched expert's U and V once (bf16)
    # plus the token activations it must move: gather (read fp32 x, write bf16 rows), GEMM1
    # reads the bf16 rows, the combine reads and writes fp32 x. The hidden H is an
    # intermediate (kept in an L2 ring by the fused kernel) and is not counted.
    alg_bytes = w_bytes + T * (4 * d + 2 * d + 2 * d + 8 * d)
    flops = 4.0 * T * d * cfg.d_ff
    peaks, peak_kind = load_peaks()
    achieved = alg_bytes / ((t_up + t_down) * 1e-3) / 1e9
    traffic = None
    prof = ROOT / "profiles" / "ffn_traffic.json"
    if prof.exists():
        try:
            traffic = json.loads(prof.read_text()).get("traffic_bytes_per_layer")
        except Exception:
            traffic = None

    # "MoE layers only" next to end-to-end -- the predictor + plan part of the
    # step captured alone and timed the same way; the MoE layers are the rest of the step
    moe_only = None
    if graph is not None:
        g_pred = pipe.capture_call(lambda sp: pipe.predict(x, sp) + pipe.plan_and_place(sp))
        for _ in range(3):
            g_pred.replay()
        torch.cuda.synchronize()
        s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s0.record()
        for _ in range(args.steps):
            g_pred.replay()
        s1.record()
        torch.cuda.synchronize()
        ms_pred = s0.elapsed_time(s1) / args.steps
        ms_moe = elapsed_ms / args.steps - ms_pred
        moe_only = {"value": T / (ms_moe * 1e-3), "unit": "tokens/s", "ms_per_step": ms_moe,
                    "ms_predictor_and_plan": ms_pred,
                    "how": "step time minus a separately captured and timed predictor + plan/place graph"}

    value = world * T * args.steps / (elapsed_ms * 1e-3)
    result = {
        "metric": METRIC,
        "value": value,
        "unit": "tokens/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": elapsed_ms / args.steps,
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "bf16",
        "data": "synthetic",
        "config": config_dict(args, world),
        "clocks": clk,
        "gpu_launches": launches,
        "roofline": {
            "kernel": ("fused grouped expert FFN (k_ffn_fused: GEMM1 relu + GEMM2 scatter-combine, H in L2 ring)"
                       if pipe.cfg.ffn == "fused" else
                       "grouped expert GEMM pair (GEMM1 relu + GEMM2 scatter-combine"
                       + (", multi-tile units k_ffn_mt)" if pipe.cfg.ffn == "mt" and args.replication != "off" else
                          ", CTA-pair cta_group::2 kernels)" if pipe.cfg.ffn == "pair" else ")")),
            "bound": "hbm",
            "achieved": achieved,
            "peak": peaks["hbm_gbs"],
            "unit": "GB/s",
            "frac": achieved / peaks["hbm_gbs"],
            "traffic": traffic,
            "peak_source": peak_kind,
            "algorithmic_bytes_per_layer": alg_bytes,
            "touched_experts_per_layer": touched,
            "ms_gemm1": t_up,
            "ms_gemm2": t_down,
            "tensor_tflops": flops / ((t_up + t_down) * 1e-3) / 1e12,
            "tensor_frac": flops / ((t_up + t_down) * 1e-3) / 1e12 / peaks["bf16_tflops_sustained"],
        },
        "checks": {"routing_exact_last_step": routing_exact, "predictor_accuracy_last_step": pred_acc},
        "moe_layers_only": moe_only,
        "cuda_graph": graph is not None or overlap is not None,
        "overlap": overlap is not None,
    }

    result["config"]["ffn_kernels"] = pipe.cfg.ffn  # resolved from --ffn auto
    if not args.no_e2e:
        pipe._bench_x, pipe._bench_graph = x, graph
        result["e2e"] = run_e2e(args, pipe, batches, world)
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cb = cpu_baseline(args)
        result["cpu_baseline"] = {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample")}
    if rank == 0:
        print(json.dumps(result))
    if world > 1:
        import torch.distributed as dist

        dist.destroy_process_group()
    return 0


def run_e2e(args, pipe, batches, world):
    """Same metric through the public pipeline with HOST buffers: pinned H2D of each batch's
    embeddings and D2H of its output stream inside the timed region. Transfers are
    double-buffered through device staging buffers on two copy streams so they overlap
    the previous/next batch's compute; the step itself runs on the fixed residual-stream
    buffer (the one whose L2 persistence window the graph was captured with)."""
    import torch

    T, d = pipe.cfg.tokens, pipe.cfg.d_model
    host_in = [b[0].cpu().pin_memory() for b in batches]
    host_out = [torch.empty(T, d, pin_memory=True) for _ in range(2)]
    st_in = [torch.empty(T, d, device="cuda") for _ in range(2)]
    st_out = [torch.empty(T, d, device="cuda") for _ in range(2)]
    x = pipe._bench_x
    h2d, d2h = torch.cuda.Stream(), torch.cuda.Stream()
    comp = torch.cuda.current_stream()
    h2d_done = [torch.cuda.Event() for _ in range(2)]
    in_free = [torch.cuda.Event() for _ in range(2)]
    comp_done = [torch.cuda.Event() for _ in range(2)]
    d2h_done = [torch.cuda.Event() for _ in range(2)]
    graph = pipe._bench_graph if not args.no_graph and getattr(pipe, "ep", None) is None else None

    def run(n, timed):
        start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        if timed:
            start.record(h2d)
        for k in range(n):
            j = k % 2
            if k >= 2:
                h2d.wait_event(in_free[j])
            with torch.cuda.stream(h2d):
                st_in[j].copy_(host_in[k % len(host_in)], non_blocking=True)
                h2d_done[j].record(h2d)
            comp.wait_event(h2d_done[j])
            x.copy_(st_in[j])
            in_free[j].record(comp)
            if graph is not None:
                graph.replay()
            else:
                pipe.step(x)
            if k >= 2:
                comp.wait_event(d2h_done[j])
            st_out[j].copy_(x)
            comp_done[j].record(comp)
            d2h.wait_event(comp_done[j])
            with torch.cuda.stream(d2h):
                host_out[j].copy_(st_out[j], non_blocking=True)
                d2h_done[j].record(d2h)
        if timed:
            end.record(d2h)
        torch.cuda.synchronize()
        return start.elapsed_time(end) if timed else 0.0

    run(args.warmup, False)
    barrier(world)
    ms = max_over_ranks(run(args.steps, True), world)
    return {"value": world * T * args.steps / (ms * 1e-3), "unit": "tokens/s",
            "h2d_bytes_per_step": T * d * 4, "d2h_bytes_per_step": T * d * 4,
            "ms_per_step": ms / args.steps,
            "api": "MoEPipeline.step over pinned host batches (H2D/D2H double-buffered through device staging "
                   "buffers on copy streams)"}


def main():
    args = parse_args()
    if args.impl == "reference":
        return run_reference(args)
    import torch

    if int(os.environ.get("WORLD_SIZE", "1")) > 1:
        torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", "0")))
    with torch.cuda.stream(torch.cuda.Stream()):  # capturable (non-legacy) compute stream
        return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
