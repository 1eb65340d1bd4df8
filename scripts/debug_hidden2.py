"""Layer-1 tcgen05 conv vs numpy conv of the GPU's own layer-0 output, under debug switches."""
import os, sys, ctypes as C
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2509_02447_b200 as q, oracle
o = oracle.Oracle()
Ws, bns, wl, bl = o.hidden_params(7, 60)
w1 = Ws[1]                       # [co][tap][ci]
g, b, m, v = bns[1]
s = (g / np.sqrt(v + np.float32(1e-5))).astype(np.float32)
wf = (w1 * s[:, None, None]).astype(np.float32)
wf = torch.tensor(wf).bfloat16().float().numpy()   # bf16 weights as the GPU uses
bias = (b - m * s).astype(np.float32)
L = q.lib()
L.qrm_hidden_debug_activation.argtypes = [C.c_void_p, C.c_void_p, C.c_int64, C.c_int, C.c_int, C.c_int64, C.c_uint64, C.c_uint64, C.c_int, C.c_void_p, C.c_void_p]
cfg = q.DetectionConfig()
imgs = q.make_corpus(cfg, 1000, 1)
def act(layer, dbg):
    os.environ["QRM_HIDDEN_DBG"] = str(dbg)
    out = torch.empty((1, 64, 64, 64), dtype=torch.bfloat16, device="cuda")
    with q.DetectionContext(cfg) as ctx:
        assert L.qrm_hidden_debug_activation(ctx._h, imgs.data_ptr(), 1, 256, 256, imgs.stride(0), 0, 7, layer, out.data_ptr(), torch.cuda.current_stream().cuda_stream) == 0
        torch.cuda.synchronize()
    return out.float().cpu().numpy()[0]
a0 = act(0, 0)
def ref_conv(x, taps):
    out = np.zeros((64, 64, 64), np.float64) + bias
    xp = np.pad(x, ((1, 1), (1, 1), (0, 0)))
    for t in taps:
        dy, dx = t // 3 - 1, t % 3 - 1
        out += np.einsum('yxc,oc->yxo', xp[1 + dy:65 + dy, 1 + dx:65 + dx], wf[:, t, :])
    return np.maximum(out, 0)
for dbg in (1, 3, 0, 2, 4, 6):
    g1 = act(1, dbg)
    taps = [4] if dbg & 1 else list(range(9))
    r = ref_conv(a0, taps)
    rel = np.linalg.norm(g1 - r) / np.linalg.norm(r)
    # per-tap attribution for the full runs: which single-tap references best explain the error
    print(f"dbg={dbg}: rel {rel:.3e}")
    if dbg in (0, 2, 4):
        err = g1 - r
        rowerr = np.linalg.norm(err, axis=(1, 2)); colerr = np.linalg.norm(err, axis=(0, 2))
        print("   worst rows", np.argsort(-rowerr)[:6], "worst cols", np.argsort(-colerr)[:6])
