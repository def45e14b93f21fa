import sys, ctypes
sys.path.insert(0, '/root/repo')
import numpy as np, torch
from paper_2605_11537_b200 import _lib
from paper_2605_11537_b200.engine import MoEPipeline, PipelineConfig
with torch.cuda.stream(torch.cuda.Stream()):
    pipe = MoEPipeline(PipelineConfig())
    b = [pipe.wl.batch(16384)[0] for _ in range(2)]
    x = torch.empty_like(b[0])
    _lib.call("mp_l2_persist", x.data_ptr(), x.numel() * 4, 1.0, torch.cuda.current_stream().cuda_stream)
    for k in range(3):
        x.copy_(b[k % 2]); pipe.step(x)
    torch.cuda.synchronize()
    lib = _lib.load_library()
    f = lib.mp_debug_router_times; f.argtypes = [ctypes.c_void_p, ctypes.c_int]
    out = np.zeros((256, 8), np.uint64)
    f(out.ctypes.data, 256)
    t = out[:128].astype(np.int64)
    base = t[:, 0].min()
    t = (t - base) / 1e3
    names = ["start", "after prologue", "first MMA", "MMA kb6", "last commit", "epi tfull", "epi done"]
    for i, n in enumerate(names):
        print(f"{n:16s} min {t[:, i].min():6.2f} med {np.median(t[:, i]):6.2f} max {t[:, i].max():6.2f}")
    t2 = (out[128:256].astype(np.int64) - base) / 1e3
    t7 = (out[:128, 7].astype(np.int64) - base) / 1e3
    print("kb6 conv: start-wait %.2f  x landed %.2f  regs read %.2f  conv done %.2f" % (np.median(t7), np.median(t2[:, 0]), np.median(t2[:, 1]), np.median(t2[:, 2])))
    print("kb6 mma: waits B from %.2f  B ok %.2f  first-MMA(kb6) %.2f" % (np.median(t2[:, 3]), np.median(t2[:, 4]), np.median(t[:, 3])))
