"""Break down the host cost of ctx.detect_device (Python side vs the C-ABI call)."""
import os, sys, time, ctypes as C
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2509_02447_b200 as q
cfg = q.DetectionConfig(); B = 4096
pool = q.make_corpus(cfg, 1000, B)
out = torch.empty((B, 24), dtype=torch.uint8, device="cuda")
def t(f, n=2000):
    f(); t0 = time.perf_counter()
    for _ in range(n): f()
    return (time.perf_counter() - t0) / n * 1e6
with q.DetectionContext(cfg) as ctx:
    L = q.lib(); h = ctx._h
    ip, op, st = pool.data_ptr(), out.data_ptr(), torch.cuda.current_stream().cuda_stream
    print("stream()", round(t(lambda: q._stream(None)), 2))
    print("current_stream", round(t(lambda: torch.cuda.current_stream().cuda_stream), 2))
    print("raw stream", round(t(lambda: torch._C._cuda_getCurrentRawStream(torch._C._cuda_getDevice())), 2))
    print("ptr+stride+shape", round(t(lambda: (pool.data_ptr(), pool.stride(0), pool.shape)), 2))
    print("count=0 call", round(t(lambda: L.qrm_detect_device(h, ip, 0, 256, 256, 196608, 0, op, st)), 2))
    torch.cuda.synchronize()
    print("full C call", round(t(lambda: L.qrm_detect_device(h, ip, B, 256, 256, 196608, 0, op, st), 400), 2))
    torch.cuda.synchronize()
    print("detect_device", round(t(lambda: ctx.detect_device(pool, 0, out=out), 400), 2))
    torch.cuda.synchronize()
