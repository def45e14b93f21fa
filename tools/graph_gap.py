"""Per-kernel overhead inside a CUDA graph: N tiny dependent kernels, replay timed with events."""
import torch

x = torch.zeros(1024, device="cuda")
s = torch.cuda.Stream()
for n in (10, 170, 500):
    with torch.cuda.stream(s):
        g = torch.cuda.CUDAGraph()
        for _ in range(3):
            x.add_(1.0)
        with torch.cuda.graph(g, stream=s):
            for _ in range(n):
                x.add_(1.0)
        g.replay()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        for _ in range(20):
            g.replay()
        b.record(s)
        torch.cuda.synchronize()
    print(f"{n} kernels: {a.elapsed_time(b) / 20 * 1e3 / n:.2f} us per kernel")
