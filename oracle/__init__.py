"""Parity oracle for the QRMark tile-detection path (TEST INFRASTRUCTURE ONLY).

Two CPU implementations live here, both loaded through ctypes:

* ``Oracle`` — ``_build/liboracle.so``, the plain-C restatement in
  ``qrmark_oracle.c`` (every function cites the reference file:line it follows).
* ``Reference`` — ``_ref/libqrmark_ref.so``, the unmodified reference core
  (``/root/reference/proj/src``) compiled in place by ``Makefile`` plus the
  ``ref_harness.cpp`` C-ABI shim.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu-baseline /
reference arm may import this package. The product never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORC_SO = os.path.join(HERE, "_build", "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libqrmark_ref.so")
REF_SRC = "/root/reference/proj"

STRATEGY = {"random": 0, "random_grid": 1, "fixed": 2}
PROFILES = {"gf16-15-12": (4, 15, 12)}


def profile_params(name: str, payload_bits: int = 48):
    """resolve_profile (rs.cpp:65-76) -> (m, n, k, t)."""
    if name == "gf16-15-12":
        return 4, 15, 12, 1
    if name == "gf256-dynamic":
        if payload_bits <= 0 or payload_bits % 8:
            raise ValueError("gf256-dynamic payload must be a positive multiple of 8 bits")
        k = payload_bits // 8
        return 8, k + 2, k, 1
    raise ValueError(f"unknown code profile: {name}")


def build(force: bool = False, ref: bool = True) -> None:
    """Compile the oracle (and the reference when its sources are present)."""
    targets = ["oracle"]
    if ref and os.path.isdir(REF_SRC):
        targets.append("ref")
    if force:
        subprocess.run(["make", "-C", HERE, "clean"], check=True, capture_output=True)
    subprocess.run(["make", "-C", HERE, "-j8", *targets], check=True, capture_output=True)


def _u8p(a):
    return a.ctypes.data_as(C.POINTER(C.c_uint8))


def _p(a, ct):
    return a.ctypes.data_as(C.POINTER(ct))


def bits_to_word(bits) -> int:
    w = 0
    for b in bits:
        w = (w << 1) | (int(b) & 1)
    return w


def word_to_bits(w: int, n: int) -> np.ndarray:
    return np.array([(w >> (n - 1 - i)) & 1 for i in range(n)], dtype=np.uint8)


class _OrcCfg(C.Structure):
    _fields_ = [("m", C.c_int), ("n", C.c_int), ("k", C.c_int), ("tile_size", C.c_int), ("strategy", C.c_int),
                ("tile_seed", C.c_uint64), ("key_seed", C.c_uint64), ("alpha", C.c_double),
                ("key_message", C.POINTER(C.c_uint8)), ("fpr", C.c_double)]


class _OrcRecord(C.Structure):
    _fields_ = [("raw", C.c_uint64), ("msg", C.c_uint64), ("decoded", C.c_int32), ("errors", C.c_int32),
                ("matches", C.c_int32), ("verified", C.c_int32), ("bit_acc", C.c_double)]


class _RefCfg(C.Structure):
    _fields_ = [("m", C.c_int), ("n", C.c_int), ("k", C.c_int), ("tile_size", C.c_int), ("strategy", C.c_int),
                ("tile_seed", C.c_uint64), ("key_seed", C.c_uint64), ("alpha", C.c_double),
                ("key_message", C.POINTER(C.c_uint8)), ("rs_workers", C.c_int), ("fpr", C.c_double),
                ("cache_enabled", C.c_int), ("cache_capacity", C.c_uint64), ("stale_after", C.c_uint64)]


class _RefRecords(C.Structure):
    _fields_ = [("raw_bits", C.POINTER(C.c_uint8)), ("has_corrected", C.POINTER(C.c_uint8)),
                ("corrected", C.POINTER(C.c_uint8)), ("errors", C.POINTER(C.c_int32)),
                ("bit_acc", C.POINTER(C.c_double)), ("verified", C.POINTER(C.c_uint8)),
                ("cache_hit", C.POINTER(C.c_uint8))]


@dataclass
class DetectCfg:
    """DetectionConfig (detect.hpp:25-37) at the reference defaults (cli.cpp:55-65)."""
    profile: str = "gf16-15-12"
    payload_bits: int = 48
    tile_size: int = 64
    strategy: str = "random_grid"
    tile_seed: int = 0
    key_seed: int = 1
    alpha: float = 0.04
    fpr: float = 1e-6
    key_message: np.ndarray | None = None  # defaults to default_message(key_seed)
    mnk: tuple | None = None  # explicit (m, n, k), overriding the profile (CodeParams::make)

    @property
    def code(self):
        if self.mnk is not None:
            m, n, k = self.mnk
            return m, n, k, (n - k) // 2
        return profile_params(self.profile, self.payload_bits)


class _Common:
    lib: C.CDLL

    def _msg(self, cfg: DetectCfg):
        m, n, k, _ = cfg.code
        if cfg.key_message is not None:
            return np.ascontiguousarray(cfg.key_message, dtype=np.uint8)
        return self.default_message(cfg.key_seed, k * m)


class Oracle(_Common):
    """ctypes view of liboracle.so (the C restatement)."""

    def __init__(self, path: str = ORC_SO):
        if not os.path.exists(path):
            build(ref=False)
        L = self.lib = C.CDLL(path)
        L.orc_rng_word.restype = C.c_uint64
        L.orc_rng_word.argtypes = [C.c_uint64] * 3
        L.orc_rng_below.restype = C.c_uint64
        L.orc_rng_below.argtypes = [C.c_uint64] * 4
        L.orc_rng_unit.restype = C.c_double
        L.orc_rng_unit.argtypes = [C.c_uint64] * 3
        L.orc_verify_threshold.argtypes = [C.c_int, C.c_double]
        L.orc_select_tile.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, C.c_uint64, C.c_uint64,
                                      C.POINTER(C.c_int), C.POINTER(C.c_int)]
        L.orc_extract.argtypes = [C.c_uint64, C.c_int, C.c_int, C.POINTER(C.c_float), C.POINTER(C.c_double)]
        L.orc_extract_exact.argtypes = [C.c_uint64, C.c_int, C.c_int, C.POINTER(C.c_uint8), C.POINTER(C.c_int64)]
        L.orc_pattern.argtypes = [C.c_uint64, C.c_int, C.c_int, C.POINTER(C.c_int8)]
        L.orc_synthetic_image.argtypes = [C.c_uint64, C.c_int, C.c_int, C.POINTER(C.c_uint8)]
        L.orc_default_message.argtypes = [C.c_uint64, C.c_int, C.POINTER(C.c_uint8)]
        L.orc_embed_grid_u8.argtypes = [C.POINTER(C.c_uint8), C.c_int, C.c_int, C.c_uint64, C.c_double, C.c_int,
                                        C.POINTER(C.c_uint8), C.c_int]
        L.orc_detect_one.argtypes = [C.POINTER(C.c_uint8), C.c_int, C.c_int, C.c_uint64, C.POINTER(_OrcCfg),
                                     C.POINTER(_OrcRecord)]
        L.orc_bw_decode_packed.argtypes = [C.c_int, C.c_int, C.c_int, C.POINTER(C.c_uint64), C.c_int64,
                                           C.POINTER(C.c_uint64), C.POINTER(C.c_int8)]
        L.orc_preprocess.argtypes = [C.POINTER(C.c_uint8), C.c_int, C.c_int, C.POINTER(C.c_float)]
        L.orc_resize_bilinear.argtypes = [C.POINTER(C.c_uint8), C.c_int, C.c_int, C.c_int, C.c_int,
                                          C.POINTER(C.c_uint8)]
        L.orc_allocate_streams.argtypes = [C.c_int, C.POINTER(C.c_double), C.POINTER(C.c_double), C.c_double,
                                           C.c_int, C.c_int, C.c_double, C.c_double, C.c_int, C.POINTER(C.c_int),
                                           C.POINTER(C.c_int), C.POINTER(C.c_double)]
        L.orc_hidden_weight.restype = C.c_float
        L.orc_hidden_weight.argtypes = [C.c_uint64, C.c_int, C.c_int, C.c_int, C.c_int]
        L.orc_hidden_bn.argtypes = [C.c_uint64, C.c_int, C.c_int] + [C.POINTER(C.c_float)] * 4
        L.orc_hidden_linear_w.restype = C.c_float
        L.orc_hidden_linear_w.argtypes = [C.c_uint64, C.c_int, C.c_int, C.c_int]
        L.orc_hidden_linear_b.restype = C.c_float
        L.orc_hidden_linear_b.argtypes = [C.c_uint64, C.c_int]
        L.orc_hidden_forward.argtypes = [C.c_uint64, C.c_int, C.c_int, C.POINTER(C.c_uint8), C.POINTER(C.c_double),
                                         C.POINTER(C.c_double)]
        L.orc_lpt_schedule.argtypes = ([C.c_int, C.POINTER(C.c_int), C.POINTER(C.c_double), C.POINTER(C.c_double),
                                        C.POINTER(C.c_int), C.c_int, C.c_double, C.c_double, C.c_int, C.c_int,
                                        C.c_int] + [C.POINTER(C.c_int)] * 3 + [C.POINTER(C.c_double)] * 2 +
                                       [C.POINTER(C.c_int)] * 2 + [C.POINTER(C.c_double), C.POINTER(C.c_int)])

    # -- learned extractor (hidden_oracle.c)
    def hidden_forward(self, seed, nbits, tile_u8):
        """fp32 conv-stack logits (double accumulation) of one l x l x 3 u8 tile."""
        t = np.ascontiguousarray(tile_u8, np.uint8)
        lg = np.zeros(nbits)
        pooled = np.zeros(nbits)
        self.lib.orc_hidden_forward(seed, nbits, t.shape[0], _u8p(t), _p(lg, C.c_double), _p(pooled, C.c_double))
        return lg, pooled

    def hidden_params(self, seed, nbits):
        """All parameters as numpy arrays (for the torch cross-check)."""
        L = self.lib
        Ws, bns = [], []
        for j in range(9):
            cin = 3 if j == 0 else 64
            cout = nbits if j == 8 else 64
            w = np.zeros((cout, 9, cin), np.float32)
            for co in range(cout):
                for t in range(9):
                    for ci in range(cin):
                        w[co, t, ci] = L.orc_hidden_weight(seed, j, co, t, ci)
            Ws.append(w)
            g, b, m, v = (C.c_float() for _ in range(4))
            bn = np.zeros((4, cout), np.float32)
            for c in range(cout):
                L.orc_hidden_bn(seed, j, c, C.byref(g), C.byref(b), C.byref(m), C.byref(v))
                bn[:, c] = (g.value, b.value, m.value, v.value)
            bns.append(bn)
        wl = np.array([[L.orc_hidden_linear_w(seed, nbits, o, i) for i in range(nbits)] for o in range(nbits)],
                      np.float32)
        bl = np.array([L.orc_hidden_linear_b(seed, o) for o in range(nbits)], np.float32)
        return Ws, bns, wl, bl

    # -- primitives
    def rng_word(self, s, st, c):
        return self.lib.orc_rng_word(s, st, c)

    def rng_below(self, s, st, c, b):
        return self.lib.orc_rng_below(s, st, c, b)

    def default_message(self, key_seed: int, n_bits: int) -> np.ndarray:
        out = np.zeros(n_bits, np.uint8)
        self.lib.orc_default_message(key_seed, n_bits, _u8p(out))
        return out

    def rs_encode(self, m, n, k, msg_bits) -> np.ndarray:
        msg = np.ascontiguousarray(msg_bits, np.uint8)
        out = np.zeros(n * m, np.uint8)
        rc = self.lib.orc_rs_encode(m, n, k, _u8p(msg), _u8p(out))
        if rc:
            raise ValueError("orc_rs_encode: invalid input")
        return out

    def bw_decode(self, m, n, k, bits):
        """-> (message bits, codeword bits, errors) or None."""
        b = np.ascontiguousarray(bits, np.uint8)
        msg = np.zeros(k * m, np.uint8)
        cw = np.zeros(n * m, np.uint8)
        e = C.c_int(0)
        rc = self.lib.orc_bw_decode(m, n, k, _u8p(b), _u8p(msg), _u8p(cw), C.byref(e))
        if rc < 0:
            raise ValueError("orc_bw_decode: invalid input")
        return (msg, cw, e.value) if rc == 1 else None

    def bw_decode_packed(self, m, n, k, words):
        w = np.ascontiguousarray(words, np.uint64)
        cw = np.zeros_like(w)
        ne = np.zeros(w.shape, np.int8)
        self.lib.orc_bw_decode_packed(m, n, k, _p(w, C.c_uint64), w.size, _p(cw, C.c_uint64), _p(ne, C.c_int8))
        return cw, ne

    def verify_threshold(self, n_bits, fpr):
        return self.lib.orc_verify_threshold(n_bits, fpr)

    def select_tile(self, w, h, l, strategy, seed, draw):
        x, y = C.c_int(), C.c_int()
        rc = self.lib.orc_select_tile(w, h, l, STRATEGY.get(strategy, strategy), seed, draw, C.byref(x), C.byref(y))
        if rc:
            raise ValueError("tile size does not fit image")
        return x.value, y.value

    def pattern(self, key_seed, bit, l):
        out = np.zeros(3 * l * l, np.int8)
        self.lib.orc_pattern(key_seed, bit, l, _p(out, C.c_int8))
        return out

    def extract(self, key_seed, n_bits, l, tile_f32):
        t = np.ascontiguousarray(tile_f32, np.float32)
        out = np.zeros(n_bits, np.float64)
        self.lib.orc_extract(key_seed, n_bits, l, _p(t, C.c_float), _p(out, C.c_double))
        return out

    def extract_exact(self, key_seed, n_bits, l, tile_u8):
        t = np.ascontiguousarray(tile_u8, np.uint8)
        out = np.zeros(n_bits, np.int64)
        self.lib.orc_extract_exact(key_seed, n_bits, l, _u8p(t), _p(out, C.c_int64))
        return out

    def synthetic_image(self, seed, w, h):
        out = np.zeros((h, w, 3), np.uint8)
        self.lib.orc_synthetic_image(seed, w, h, _u8p(out))
        return out

    def embed_grid(self, img, key_seed, alpha, l, cw_bits):
        im = np.ascontiguousarray(img, np.uint8).copy()
        bits = np.ascontiguousarray(cw_bits, np.uint8)
        self.lib.orc_embed_grid_u8(_u8p(im), im.shape[1], im.shape[0], key_seed, alpha, l, _u8p(bits), bits.size)
        return im

    def make_corpus(self, first_seed, count, w, h, cfg: DetectCfg = DetectCfg(), embed=True):
        m, n, k, _ = cfg.code
        cw = self.rs_encode(m, n, k, self._msg(cfg))
        out = np.zeros((count, h, w, 3), np.uint8)
        for i in range(count):
            img = self.synthetic_image(first_seed + i, w, h)
            out[i] = self.embed_grid(img, cfg.key_seed, cfg.alpha, cfg.tile_size, cw) if embed else img
        return out

    def preprocess(self, img):
        im = np.ascontiguousarray(img, np.uint8)
        out = np.zeros((256, 256, 3), np.float32)
        self.lib.orc_preprocess(_u8p(im), im.shape[1], im.shape[0], _p(out, C.c_float))
        return out

    def resize_bilinear(self, img, ow, oh):
        im = np.ascontiguousarray(img, np.uint8)
        out = np.zeros((oh, ow, 3), np.uint8)
        self.lib.orc_resize_bilinear(_u8p(im), im.shape[1], im.shape[0], ow, oh, _u8p(out))
        return out

    def detect(self, images, cfg: DetectCfg = DetectCfg(), first_draw: int = 0):
        """detect_one over images with draw_index = first_draw + i. Returns a dict of arrays."""
        m, n, k, _ = cfg.code
        msg = self._msg(cfg)
        c = _OrcCfg(m, n, k, cfg.tile_size, STRATEGY[cfg.strategy], cfg.tile_seed, cfg.key_seed, cfg.alpha,
                    _u8p(msg), cfg.fpr)
        recs = []
        for i, img in enumerate(images):
            im = np.ascontiguousarray(img, np.uint8)
            r = _OrcRecord()
            rc = self.lib.orc_detect_one(_u8p(im), im.shape[1], im.shape[0], first_draw + i, C.byref(c), C.byref(r))
            if rc:
                raise ValueError("orc_detect_one failed")
            recs.append((r.raw, r.msg, r.decoded, r.errors, r.matches, r.verified, r.bit_acc))
        a = np.array(recs, dtype=object).reshape(-1, 7)
        return {"raw": a[:, 0].astype(np.uint64), "msg": a[:, 1].astype(np.uint64),
                "decoded": a[:, 2].astype(np.int32), "errors": a[:, 3].astype(np.int32),
                "matches": a[:, 4].astype(np.int32), "verified": a[:, 5].astype(np.int32),
                "bit_acc": a[:, 6].astype(np.float64)}

    def allocate_streams(self, time, memory, b0, B, P, m_cap, eps, stall_cap):
        K = len(time)
        t = np.ascontiguousarray(time, np.float64)
        u = np.ascontiguousarray(memory, np.float64)
        s = np.zeros(K, np.int32)
        mb = np.zeros(K, np.int32)
        bn = C.c_double()
        rc = self.lib.orc_allocate_streams(K, _p(t, C.c_double), _p(u, C.c_double), b0, B, P, m_cap, eps, stall_cap,
                                           _p(s, C.c_int), _p(mb, C.c_int), C.byref(bn))
        return rc, s.tolist(), mb.tolist(), bn.value

    def lpt_schedule(self, ids, lat, mem, units, S, lam, m_cap, b_min, B):
        return _lpt(self.lib.orc_lpt_schedule, ids, lat, mem, units, S, lam, m_cap, b_min, B)


def _lpt(fn, ids, lat, mem, units, S, lam, m_cap, b_min, B):
    n = len(ids)
    ids_ = np.ascontiguousarray(ids, np.int32)
    lat_ = np.ascontiguousarray(lat, np.float64)
    mem_ = np.ascontiguousarray(mem, np.float64)
    un_ = np.ascontiguousarray(units, np.int32)
    cap = int(un_.sum()) + n + 1
    ps, pi, pu, pm = (np.zeros(cap, np.int32) for _ in range(4))
    pl, pme = np.zeros(cap), np.zeros(cap)
    npieces, mu = C.c_int(), C.c_int()
    loads = np.zeros(S)
    rc = fn(n, _p(ids_, C.c_int), _p(lat_, C.c_double), _p(mem_, C.c_double), _p(un_, C.c_int), S, lam, m_cap,
            b_min, B, cap, _p(ps, C.c_int), _p(pi, C.c_int), _p(pu, C.c_int), _p(pl, C.c_double),
            _p(pme, C.c_double), _p(pm, C.c_int), C.byref(npieces), _p(loads, C.c_double), C.byref(mu))
    if rc:
        return rc, None
    c = npieces.value
    pieces = list(zip(ps[:c].tolist(), pi[:c].tolist(), pu[:c].tolist(), pl[:c].tolist(), pme[:c].tolist(),
                      pm[:c].tolist()))
    return 0, {"pieces": pieces, "loads": loads.tolist(), "m_unit": mu.value}


class Reference(_Common):
    """ctypes view of the compiled reference (oracle/_ref/libqrmark_ref.so)."""

    @staticmethod
    def available() -> bool:
        return os.path.exists(REF_SO) or os.path.isdir(REF_SRC)

    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            if not os.path.isdir(REF_SRC):
                raise FileNotFoundError("reference library not built and sources absent")
            build(ref=True)
        L = self.lib = C.CDLL(path)
        L.ref_last_error.restype = C.c_char_p
        L.ref_default_message.argtypes = [C.c_uint64, C.c_int, C.POINTER(C.c_uint8)]
        L.ref_rng_word.restype = C.c_uint64
        L.ref_rng_word.argtypes = [C.c_uint64] * 3
        L.ref_rng_below.restype = C.c_uint64
        L.ref_rng_below.argtypes = [C.c_uint64] * 4
        L.ref_bw_decode_packed.restype = C.c_int64
        L.ref_bw_decode_packed.argtypes = [C.c_int, C.c_int, C.c_int, C.POINTER(C.c_uint64), C.c_int64, C.c_int,
                                           C.POINTER(C.c_uint64), C.POINTER(C.c_int8)]
        L.ref_bw_decode_symbols.argtypes = [C.c_int, C.c_int, C.c_int, C.POINTER(C.c_uint8), C.c_int64,
                                            C.POINTER(C.c_uint8), C.POINTER(C.c_int8)]
        L.ref_bw_decode_symbols_mt.restype = C.c_int64
        L.ref_bw_decode_symbols_mt.argtypes = [C.c_int, C.c_int, C.c_int, C.POINTER(C.c_uint8), C.c_int64, C.c_int,
                                               C.POINTER(C.c_uint8), C.POINTER(C.c_int8)]
        L.ref_verify_threshold.argtypes = [C.c_int, C.c_double, C.POINTER(C.c_int)]
        L.ref_synthetic_image.argtypes = [C.c_uint64, C.c_int, C.c_int, C.POINTER(C.c_uint8)]
        L.ref_make_corpus.argtypes = [C.c_uint64, C.c_int64, C.c_int, C.c_int, C.c_uint64, C.c_double, C.c_int,
                                      C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.POINTER(C.c_uint8)]
        L.ref_preprocess.argtypes = [C.POINTER(C.c_uint8), C.c_int, C.c_int, C.c_int, C.POINTER(C.c_float)]
        L.ref_resize_bilinear.argtypes = [C.POINTER(C.c_uint8), C.c_int, C.c_int, C.c_int, C.c_int,
                                          C.POINTER(C.c_uint8)]
        L.ref_select_tile.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, C.c_uint64, C.c_uint64,
                                      C.POINTER(C.c_int), C.POINTER(C.c_int)]
        L.ref_extract.argtypes = [C.c_uint64, C.c_int, C.c_double, C.c_int, C.POINTER(C.c_float),
                                  C.POINTER(C.c_double)]
        L.ref_pattern.argtypes = [C.c_uint64, C.c_int, C.c_int, C.c_int, C.POINTER(C.c_int8)]
        L.ref_detect_sequential.argtypes = [C.POINTER(C.POINTER(C.c_uint8)), C.POINTER(C.c_int),
                                            C.POINTER(C.c_int), C.c_int64, C.c_uint64, C.POINTER(_RefCfg),
                                            C.POINTER(_RefRecords)]
        L.ref_read_ppm.argtypes = [C.c_char_p, C.POINTER(C.c_uint8), C.c_int64, C.POINTER(C.c_int), C.POINTER(C.c_int)]
        L.ref_write_ppm.argtypes = [C.c_char_p, C.POINTER(C.c_uint8), C.c_int, C.c_int]
        L.ref_apply_attack.argtypes = [C.POINTER(C.c_uint8), C.c_int, C.c_int, C.c_char_p, C.c_double, C.c_void_p,
                                       C.c_int64, C.POINTER(C.c_int), C.POINTER(C.c_int), C.POINTER(C.c_int)]
        L.ref_detect_json.restype = C.c_int64
        L.ref_detect_json.argtypes = [C.POINTER(C.POINTER(C.c_uint8)), C.POINTER(C.c_int), C.POINTER(C.c_int),
                                      C.c_int64, C.POINTER(_RefCfg), C.c_char_p, C.c_int64]
        L.ref_detect_batch.restype = C.c_int64
        L.ref_detect_batch.argtypes = [C.POINTER(C.POINTER(C.c_uint8)), C.POINTER(C.c_int), C.POINTER(C.c_int),
                                       C.c_int64, C.POINTER(_RefCfg), C.POINTER(C.c_int), C.POINTER(C.c_int),
                                       C.POINTER(_RefRecords)]
        L.ref_allocate_streams.argtypes = [C.c_int, C.POINTER(C.c_double), C.POINTER(C.c_double), C.c_double,
                                           C.c_int, C.c_int, C.c_double, C.c_double, C.c_int, C.POINTER(C.c_int),
                                           C.POINTER(C.c_int), C.POINTER(C.c_double)]
        L.ref_lpt_schedule.argtypes = ([C.c_int, C.POINTER(C.c_int), C.POINTER(C.c_double), C.POINTER(C.c_double),
                                        C.POINTER(C.c_int), C.c_int, C.c_double, C.c_double, C.c_int, C.c_int,
                                        C.c_int] + [C.POINTER(C.c_int)] * 3 + [C.POINTER(C.c_double)] * 2 +
                                       [C.POINTER(C.c_int)] * 2 + [C.POINTER(C.c_double), C.POINTER(C.c_int)])
        L.ref_measure_stages_scripted.argtypes = [C.c_int, C.c_int, C.c_double, C.POINTER(C.c_int64),
                                                  C.POINTER(C.c_double), C.POINTER(C.c_double),
                                                  C.POINTER(C.c_double), C.POINTER(C.c_double)]

    def last_error(self) -> str:
        return self.lib.ref_last_error().decode()

    def rng_word(self, s, st, c):
        return self.lib.ref_rng_word(s, st, c)

    def rng_below(self, s, st, c, b):
        return self.lib.ref_rng_below(s, st, c, b)

    def default_message(self, key_seed, n_bits):
        out = np.zeros(n_bits, np.uint8)
        self.lib.ref_default_message(key_seed, n_bits, _u8p(out))
        return out

    def rs_encode(self, m, n, k, msg_bits):
        msg = np.ascontiguousarray(msg_bits, np.uint8)
        out = np.zeros(n * m, np.uint8)
        if self.lib.ref_rs_encode(m, n, k, _u8p(msg), _u8p(out)):
            raise ValueError(self.last_error())
        return out

    def bw_decode(self, m, n, k, bits):
        b = np.ascontiguousarray(bits, np.uint8)
        msg = np.zeros(k * m, np.uint8)
        cw = np.zeros(n * m, np.uint8)
        e = C.c_int(0)
        rc = self.lib.ref_bw_decode(m, n, k, _u8p(b), _u8p(msg), _u8p(cw), C.byref(e))
        if rc < 0:
            raise ValueError(self.last_error())
        return (msg, cw, e.value) if rc == 1 else None

    def bw_decode_packed(self, m, n, k, words, threads=1):
        w = np.ascontiguousarray(words, np.uint64)
        cw = np.zeros_like(w)
        ne = np.zeros(w.shape, np.int8)
        wall = self.lib.ref_bw_decode_packed(m, n, k, _p(w, C.c_uint64), w.size, threads, _p(cw, C.c_uint64),
                                             _p(ne, C.c_int8))
        if wall < 0:
            raise ValueError(self.last_error())
        return cw, ne, wall

    def bw_decode_symbols_mt(self, m, n, k, recv, threads=1):
        """bw_decode over symbol rows on `threads` host threads -> (cw, nerr, wall_ns)."""
        r = np.ascontiguousarray(recv, np.uint8).reshape(-1, n)
        cw = np.zeros_like(r)
        ne = np.zeros(r.shape[0], np.int8)
        wall = self.lib.ref_bw_decode_symbols_mt(m, n, k, _u8p(r), r.shape[0], threads, _u8p(cw), _p(ne, C.c_int8))
        if wall < 0:
            raise ValueError(self.last_error())
        return cw, ne, wall

    def bw_decode_symbols(self, m, n, k, recv):
        r = np.ascontiguousarray(recv, np.uint8).reshape(-1, n)
        cw = np.zeros_like(r)
        ne = np.zeros(r.shape[0], np.int8)
        if self.lib.ref_bw_decode_symbols(m, n, k, _u8p(r), r.shape[0], _u8p(cw), _p(ne, C.c_int8)):
            raise ValueError(self.last_error())
        return cw, ne

    def verify_threshold(self, n_bits, fpr):
        t = C.c_int()
        if self.lib.ref_verify_threshold(n_bits, fpr, C.byref(t)):
            raise ValueError(self.last_error())
        return t.value

    def synthetic_image(self, seed, w, h):
        out = np.zeros((h, w, 3), np.uint8)
        self.lib.ref_synthetic_image(seed, w, h, _u8p(out))
        return out

    def make_corpus(self, first_seed, count, w, h, cfg: DetectCfg = DetectCfg(), embed=True, threads=None):
        m, n, k, _ = cfg.code
        out = np.zeros((count, h, w, 3), np.uint8)
        threads = threads or os.cpu_count() or 1
        if self.lib.ref_make_corpus(first_seed, count, w, h, cfg.key_seed, cfg.alpha, m, n, k, cfg.tile_size,
                                    int(embed), threads, _u8p(out)):
            raise ValueError(self.last_error())
        return out

    def preprocess(self, img, fused=False):
        im = np.ascontiguousarray(img, np.uint8)
        out = np.zeros((256, 256, 3), np.float32)
        if self.lib.ref_preprocess(_u8p(im), im.shape[1], im.shape[0], int(fused), _p(out, C.c_float)):
            raise ValueError(self.last_error())
        return out

    def resize_bilinear(self, img, ow, oh):
        im = np.ascontiguousarray(img, np.uint8)
        out = np.zeros((oh, ow, 3), np.uint8)
        self.lib.ref_resize_bilinear(_u8p(im), im.shape[1], im.shape[0], ow, oh, _u8p(out))
        return out

    def select_tile(self, w, h, l, strategy, seed, draw):
        x, y = C.c_int(), C.c_int()
        if self.lib.ref_select_tile(w, h, l, STRATEGY.get(strategy, strategy), seed, draw, C.byref(x), C.byref(y)):
            raise ValueError(self.last_error())
        return x.value, y.value

    def extract(self, key_seed, n_bits, alpha, l, tile_f32):
        t = np.ascontiguousarray(tile_f32, np.float32)
        out = np.zeros(n_bits)
        if self.lib.ref_extract(key_seed, n_bits, alpha, l, _p(t, C.c_float), _p(out, C.c_double)):
            raise ValueError(self.last_error())
        return out

    def pattern(self, key_seed, n_bits, l, bit):
        out = np.zeros(3 * l * l, np.int8)
        self.lib.ref_pattern(key_seed, n_bits, l, bit, _p(out, C.c_int8))
        return out

    def _cfg(self, cfg: DetectCfg, rs_workers=32, cache=True, cache_capacity=4096, stale_after=1 << 20):
        m, n, k, _ = cfg.code
        msg = self._msg(cfg)
        c = _RefCfg(m, n, k, cfg.tile_size, STRATEGY[cfg.strategy], cfg.tile_seed, cfg.key_seed, cfg.alpha,
                    _u8p(msg), rs_workers, cfg.fpr, int(cache), cache_capacity, stale_after)
        return c, msg

    def _records(self, count, cfg: DetectCfg):
        m, n, k, _ = cfg.code
        arrs = {"raw_bits": np.zeros((count, n * m), np.uint8), "has_corrected": np.zeros(count, np.uint8),
                "corrected": np.zeros((count, k * m), np.uint8), "errors": np.zeros(count, np.int32),
                "bit_acc": np.zeros(count), "verified": np.zeros(count, np.uint8),
                "cache_hit": np.zeros(count, np.uint8)}
        r = _RefRecords(_u8p(arrs["raw_bits"]), _u8p(arrs["has_corrected"]), _u8p(arrs["corrected"]),
                        _p(arrs["errors"], C.c_int32), _p(arrs["bit_acc"], C.c_double), _u8p(arrs["verified"]),
                        _u8p(arrs["cache_hit"]))
        return r, arrs

    @staticmethod
    def _imgs(images):
        keep = [np.ascontiguousarray(im, np.uint8) for im in images]
        ptrs = (C.POINTER(C.c_uint8) * len(keep))(*[_u8p(a) for a in keep])
        ws = (C.c_int * len(keep))(*[a.shape[1] for a in keep])
        hs = (C.c_int * len(keep))(*[a.shape[0] for a in keep])
        return keep, ptrs, ws, hs

    def detect_sequential(self, images, cfg: DetectCfg = DetectCfg(), first_draw=0, cache=True):
        keep, ptrs, ws, hs = self._imgs(images)
        c, msg = self._cfg(cfg, cache=cache)
        r, arrs = self._records(len(keep), cfg)
        if self.lib.ref_detect_sequential(ptrs, ws, hs, len(keep), first_draw, C.byref(c), C.byref(r)):
            raise ValueError(self.last_error())
        return arrs

    def read_ppm(self, path):
        """read_ppm (image.cpp:129-146) -> uint8 [H, W, 3]; ValueError carries the reference's message."""
        w, h = C.c_int(), C.c_int()
        p = os.fsencode(path)
        if self.lib.ref_read_ppm(p, None, 0, C.byref(w), C.byref(h)):
            raise ValueError(self.last_error())
        out = np.empty((h.value, w.value, 3), np.uint8)
        if self.lib.ref_read_ppm(p, _u8p(out), out.nbytes, C.byref(w), C.byref(h)):
            raise ValueError(self.last_error())
        return out

    def write_ppm(self, img, path):
        img = np.ascontiguousarray(img, np.uint8)
        if self.lib.ref_write_ppm(os.fsencode(path), _u8p(img), img.shape[1], img.shape[0]):
            raise ValueError(self.last_error())

    def apply_attack(self, img, op: str, param: float):
        """apply_attack (transforms.cpp:289-362) -> uint8 [H', W', 3] (float32 for normalize)."""
        img = np.ascontiguousarray(img, np.uint8)
        ow, oh, fl = C.c_int(), C.c_int(), C.c_int()
        args = (_u8p(img), img.shape[1], img.shape[0], op.encode(), float(param))
        if self.lib.ref_apply_attack(*args, None, 0, C.byref(ow), C.byref(oh), C.byref(fl)):
            raise ValueError(self.last_error())
        out = np.empty((oh.value, ow.value, 3), np.float32 if fl.value else np.uint8)
        if self.lib.ref_apply_attack(*args, out.ctypes.data, out.nbytes, C.byref(ow), C.byref(oh), C.byref(fl)):
            raise ValueError(self.last_error())
        return out

    def detect_json(self, images, cfg: DetectCfg = DetectCfg(), rs_workers: int = 1, cache: bool = True,
                    cache_capacity: int = 4096, stale_after: int = 1 << 20) -> str:
        """cmd_detect's records array: detect_batch + record_to_json(deterministic) + dump(2).
        rs_workers = 1 makes the codebook's hit order deterministic (index order)."""
        keep, ptrs, ws, hs = self._imgs(images)
        c, msg = self._cfg(cfg, rs_workers=rs_workers, cache=cache, cache_capacity=cache_capacity,
                           stale_after=stale_after)
        n = self.lib.ref_detect_json(ptrs, ws, hs, len(keep), C.byref(c), None, 0)
        if n < 0:
            raise ValueError(self.last_error())
        buf = C.create_string_buffer(n + 1)
        self.lib.ref_detect_json(ptrs, ws, hs, len(keep), C.byref(c), buf, n + 1)
        return buf.value.decode()

    def detect_batch(self, images, cfg: DetectCfg = DetectCfg(), plan=None, rs_workers=32, records=True):
        """detect_batch (detect.cpp:250) -> (records or None, wall_ns)."""
        keep, ptrs, ws, hs = self._imgs(images)
        c, msg = self._cfg(cfg, rs_workers=rs_workers)
        r, arrs = self._records(len(keep), cfg) if records else (None, None)
        if plan is not None:
            s3 = (C.c_int * 3)(*plan[0])
            m3 = (C.c_int * 3)(*plan[1])
        else:
            s3 = m3 = None
        wall = self.lib.ref_detect_batch(ptrs, ws, hs, len(keep), C.byref(c), s3, m3,
                                         C.byref(r) if r is not None else None)
        if wall < 0:
            raise ValueError(self.last_error())
        return arrs, wall

    def allocate_streams(self, time, memory, b0, B, P, m_cap, eps, stall_cap):
        K = len(time)
        t = np.ascontiguousarray(time, np.float64)
        u = np.ascontiguousarray(memory, np.float64)
        s = np.zeros(K, np.int32)
        mb = np.zeros(K, np.int32)
        bn = C.c_double()
        rc = self.lib.ref_allocate_streams(K, _p(t, C.c_double), _p(u, C.c_double), b0, B, P, m_cap, eps, stall_cap,
                                           _p(s, C.c_int), _p(mb, C.c_int), C.byref(bn))
        return rc, s.tolist(), mb.tolist(), bn.value

    def lpt_schedule(self, ids, lat, mem, units, S, lam, m_cap, b_min, B):
        return _lpt(self.lib.ref_lpt_schedule, ids, lat, mem, units, S, lam, m_cap, b_min, B)

    def measure_stages_scripted(self, iters, b0, clock_values, mem, prep_share):
        K = len(mem)
        cv = np.ascontiguousarray(clock_values, np.int64)
        m_ = np.ascontiguousarray(mem, np.float64)
        p_ = np.ascontiguousarray(prep_share, np.float64)
        t_out, p_out = np.zeros(K), np.zeros(K)
        rc = self.lib.ref_measure_stages_scripted(K, iters, b0, _p(cv, C.c_int64), _p(m_, C.c_double),
                                                  _p(p_, C.c_double), _p(t_out, C.c_double), _p(p_out, C.c_double))
        return rc, t_out.tolist(), p_out.tolist()
