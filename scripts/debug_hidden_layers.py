"""Per-layer check of the tcgen05 conv stack: each layer's GPU output vs a
float64 conv of the GPU's own previous-layer output (bf16 weights as the GPU
uses them), so a layer's own error is isolated from the error it inherits."""
import os, sys, ctypes as C
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2509_02447_b200 as q, oracle
o = oracle.Oracle()
SEED, NB = 7, 60
Ws, bns, wl, bl = o.hidden_params(SEED, NB)
L = q.lib()
L.qrm_hidden_debug_activation.argtypes = [C.c_void_p, C.c_void_p, C.c_int64, C.c_int, C.c_int, C.c_int64,
                                          C.c_uint64, C.c_uint64, C.c_int, C.c_void_p, C.c_void_p]
cfg = q.DetectionConfig()
NT = int(sys.argv[1]) if len(sys.argv) > 1 else 2
imgs = torch.cat([q.make_corpus(cfg, 1000, NT // 2), q.make_corpus(cfg, 5000, NT - NT // 2, embed=False)])
host = imgs.cpu().numpy()

def act(layer):
    if layer == 8:
        out = torch.empty((NT, 32, 64), dtype=torch.float32, device="cuda")
    else:
        out = torch.empty((NT, 64, 64, 64), dtype=torch.bfloat16, device="cuda")
    with q.DetectionContext(cfg) as ctx:
        assert L.qrm_hidden_debug_activation(ctx._h, imgs.data_ptr(), NT, 256, 256, imgs.stride(0), 0, SEED, layer,
                                             out.data_ptr(), torch.cuda.current_stream().cuda_stream) == 0
        torch.cuda.synchronize()
    return out.float().cpu().numpy().astype(np.float64)

def folded(j, bf16):
    w = Ws[j]
    g, b, m, v = bns[j]
    s = (g / np.sqrt(v + np.float32(1e-5))).astype(np.float32)
    wf = (w * s[:, None, None]).astype(np.float32)
    if bf16:
        wf = torch.tensor(wf).bfloat16().float().numpy()
    return wf.astype(np.float64), (b - m * s).astype(np.float32).astype(np.float64)

def conv(x, wf, bias):
    cout = wf.shape[0]
    out = np.zeros((64, 64, cout)) + bias
    xp = np.pad(x, ((1, 1), (1, 1), (0, 0)))
    for t in range(9):
        dy, dx = t // 3 - 1, t % 3 - 1
        out += np.einsum('yxc,oc->yxo', xp[1 + dy:65 + dy, 1 + dx:65 + dx], wf[:, t, :])
    return np.maximum(out, 0)

prev = None
for j in range(9):
    g = act(j)
    for i in range(NT):
        if j == 0:
            x0, y0 = o.select_tile(256, 256, 64, "random_grid", 0, i)
            tile = host[i, y0:y0 + 64, x0:x0 + 64].astype(np.float64)
            xin = (tile / 127.5 - 1.0).astype(np.float32).astype(np.float64)
        else:
            xin = prev[i]
        wf, bias = folded(j, bf16=(j > 0))
        r = conv(xin, wf, bias)
        if j == 8:
            rs = r.reshape(32, 128, -1).sum(axis=1)  # per-block channel sums
            gg = g[i][:, :rs.shape[1]]
            rel = np.linalg.norm(gg - rs) / np.linalg.norm(rs)
            print(f"layer {j} tile {i}: pool rel {rel:.3e}")
        else:
            rb = torch.tensor(r).bfloat16().double().numpy()
            err = g[i] - rb
            rel = np.linalg.norm(err) / np.linalg.norm(rb)
            rowerr = np.linalg.norm(err, axis=(1, 2)); colerr = np.linalg.norm(err, axis=(0, 2))
            print(f"layer {j} tile {i}: rel {rel:.3e} worst rows {np.argsort(-rowerr)[:4]} {rowerr[np.argsort(-rowerr)[:4]].round(2)} "
                  f"worst cols {np.argsort(-colerr)[:4]}", flush=True)
    prev = g
