"""Per-layer parity of the conv extractor vs the fp32 oracle (diagnostics)."""
import os, sys, ctypes as C
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2509_02447_b200 as q, oracle
o = oracle.Oracle()
o.lib.orc_hidden_activation.argtypes = [C.c_uint64, C.c_int, C.c_int, C.POINTER(C.c_uint8), C.c_int, C.POINTER(C.c_float)]
L = q.lib()
L.qrm_hidden_debug_activation.argtypes = [C.c_void_p, C.c_void_p, C.c_int64, C.c_int, C.c_int, C.c_int64, C.c_uint64, C.c_uint64, C.c_int, C.c_void_p, C.c_void_p]
cfg = q.DetectionConfig()
imgs = q.make_corpus(cfg, 1000, 2)
host = imgs.cpu().numpy()
with q.DetectionContext(cfg) as ctx:
    for layer in range(0, 9):
        n = 2
        if layer < 8:
            out = torch.empty((n, 64, 64, 64), dtype=torch.bfloat16, device="cuda")
        else:
            out = torch.empty((n, 32, 64), dtype=torch.float32, device="cuda")
        rc = L.qrm_hidden_debug_activation(ctx._h, imgs.data_ptr(), n, 256, 256, imgs.stride(0), 0, 7, layer, out.data_ptr(), torch.cuda.current_stream().cuda_stream)
        assert rc == 0, L.qrm_last_error()
        torch.cuda.synchronize()
        g = out.float().cpu().numpy()
        for i in range(n):
            x, y = o.select_tile(256, 256, 64, "random_grid", 0, i)
            tile = np.ascontiguousarray(host[i, y:y+64, x:x+64])
            cout = 60 if layer == 8 else 64
            ref = np.zeros(64 * 64 * cout, np.float32)
            o.lib.orc_hidden_activation(7, 60, 64, tile.ctypes.data_as(C.POINTER(C.c_uint8)), layer, ref.ctypes.data_as(C.POINTER(C.c_float)))
            ref = ref.reshape(64, 64, cout)
            if layer < 8:
                gi = g[i]
                err = np.abs(gi - ref)
                rel = np.linalg.norm(gi - ref) / max(1e-9, np.linalg.norm(ref))
                bad = np.argwhere(err > 0.05 * (np.abs(ref) + 0.1))
                print(f"layer {layer} img {i}: rel {rel:.3e} maxerr {err.max():.3e} nbad {len(bad)} first bad {bad[:5].tolist()}")
                if len(bad) and layer <= 2 and i == 0:
                    for (py, px, c) in bad[:8]:
                        print("   ", py, px, c, "gpu", gi[py, px, c], "ref", ref[py, px, c])
            else:
                gs = g[i].reshape(32, 64)[:, :60].sum(0)
                rs = ref.reshape(-1, 60).sum(0)
                print(f"pool img {i}: rel {np.linalg.norm(gs-rs)/np.linalg.norm(rs):.3e}", gs[:4], rs[:4])
