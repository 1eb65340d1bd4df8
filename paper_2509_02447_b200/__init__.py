"""B200-native QRMark tile-detection path (arXiv 2509.02447), Python host layer.

A thin ctypes layer over the C-ABI in ``include/qrmark_gpu.h`` (library
``_lib/libqrmark_b200.so``, hand-written sm_100a kernels). Names follow the
reference C++ API in ``proj/include/qrmark`` (``resolve_profile``,
``DetectionConfig``, ``DetectionContext``, ``detect_batch``, ``bw_decode``,
``allocate_streams``, ``lpt_schedule``, ``warmup_profile``) so code written
against the reference reads the same. There is no CPU fallback: importing
works without a GPU, but every compute call needs the CUDA library and a
device and raises ``QrmError`` otherwise.

Torch is used only as plumbing (device buffers and streams): any call that
takes device memory accepts a CUDA ``torch.Tensor`` and runs on the current
torch stream.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "_lib", "libqrmark_b200.so")

# Exported symbols of include/qrmark_gpu.h (checked by the CPU test suite).
ABI_SYMBOLS = (
    "qrm_last_error", "qrm_abi_version", "qrm_device_count", "qrm_ctx_create", "qrm_ctx_destroy", "qrm_ctx_info",
    "qrm_ctx_set_extractor", "qrm_ppm_read", "qrm_ppm_write", "qrm_ppm_read_batch", "qrm_records_json", "qrm_cache_hits", "qrm_attack_device", "qrm_warmup_profile_mode", "qrm_extract_tiles_device", "qrm_detect_host_multi", "qrm_detect_host_lpt", "qrm_ctx_set_transfer_split",
    "qrm_detect_device", "qrm_detect_host", "qrm_detect_ragged", "qrm_extract_device", "qrm_preprocess_host",
    "qrm_rs_decode_packed_device", "qrm_rs_decode_symbols_device", "qrm_rs_stress_device", "qrm_rs_stress_symbols_device", "qrm_rs_codebook_clear", "qrm_rs_encode_packed",
    "qrm_verify_threshold", "qrm_make_corpus_device", "qrm_patterns_device", "qrm_allocate_streams",
    "qrm_lpt_schedule", "qrm_warmup_profile", "qrm_ctx_set_plan", "qrm_kernel_launch_count",
    "qrm_probe_decode_kernel", "qrm_resample_host", "qrm_extract_float_host", "qrm_hidden_detect_device",
    "qrm_ctx_set_input_overlap", "qrm_hidden_debug_activation", "qrm_warmup_saturation", "qrm_allocate_streams_sat", "qrm_device_cpus", "qrm_detect_host_timed", "qrm_detect_host_images",
)


class QrmError(RuntimeError):
    """Base of the mapped status codes."""


class InvalidInput(QrmError, ValueError):
    """qrmark::InvalidInput (errors.hpp:11)."""


class DivisionByZero(QrmError, ArithmeticError):
    """qrmark::DivisionByZero (errors.hpp:16)."""


class InfeasibleConfig(QrmError):
    """qrmark::InfeasibleConfig (errors.hpp:22)."""


class CudaError(QrmError):
    pass


_STATUS = {1: InvalidInput, 2: DivisionByZero, 3: InfeasibleConfig, 4: CudaError, 5: CudaError, 6: QrmError}

RECORD_DTYPE = np.dtype([("raw", "<u8"), ("msg", "<u8"), ("status", "u1"), ("errors", "u1"), ("matches", "u1"),
                         ("verified", "u1"), ("ties", "u1"), ("reserved", "u1", (3,))])
assert RECORD_DTYPE.itemsize == 24

TILE_STRATEGY = {"random": 0, "random_grid": 1, "fixed": 2}
EXTRACTOR = {"spread_spectrum": 0, "conv": 1}  # QRM_EXTRACTOR_*


class _Config(C.Structure):
    _fields_ = [("symbol_bits", C.c_int), ("n", C.c_int), ("k", C.c_int), ("tile_size", C.c_int),
                ("tile_strategy", C.c_int), ("tile_seed", C.c_uint64), ("key_seed", C.c_uint64),
                ("alpha", C.c_double), ("key_message", C.POINTER(C.c_uint8)), ("fpr_target", C.c_double)]


class _Plan(C.Structure):
    _fields_ = [("streams", C.c_int * 3), ("minibatch", C.c_int * 3)]


class _StageLoad(C.Structure):
    _fields_ = [("ns", C.c_int64 * 3)]


class _StageTimes(C.Structure):
    _fields_ = [("wall_ns", C.c_int64), ("busy_ns", C.c_int64 * 3), ("image_ns", C.c_void_p)]


class _HostStats(C.Structure):
    _fields_ = [("wall_ms", C.c_double), ("h2d_bytes", C.c_double), ("d2h_bytes", C.c_double),
                ("minibatches", C.c_int), ("kernel_launches", C.c_int)]


_lib = None


def lib() -> C.CDLL:
    """Load the native library (raises if it was not built — no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise QrmError(f"native library missing: {LIB_PATH} (run python -m paper_2509_02447_b200.build)")
        L = C.CDLL(LIB_PATH)
        vp, i64, u64, i32 = C.c_void_p, C.c_int64, C.c_uint64, C.c_int
        L.qrm_last_error.restype = C.c_char_p
        L.qrm_kernel_launch_count.restype = u64
        L.qrm_ctx_create.argtypes = [i32, C.POINTER(_Config), C.POINTER(vp)]
        L.qrm_ctx_destroy.argtypes = [vp]
        L.qrm_ctx_info.argtypes = [vp, C.POINTER(u64), C.POINTER(u64), C.POINTER(i32), C.POINTER(i32)]
        L.qrm_ctx_set_extractor.argtypes = [vp, i32, u64]
        L.qrm_ctx_set_transfer_split.argtypes = [vp, C.c_double]
        L.qrm_ctx_set_input_overlap.argtypes = [vp, i32]
        L.qrm_detect_host_timed.argtypes = [vp, vp, i64, i32, i32, i64, u64, vp, C.POINTER(_Plan), i32,
                                            C.POINTER(_StageLoad), C.POINTER(_StageTimes)]
        L.qrm_detect_host_images.argtypes = [vp, C.POINTER(vp), i64, i32, i32, u64, vp, C.POINTER(_Plan),
                                             C.POINTER(_StageLoad), C.POINTER(_StageTimes)]
        L.qrm_hidden_debug_activation.argtypes = [vp, vp, i64, i32, i32, i64, u64, u64, i32, vp, vp]
        L.qrm_detect_host_lpt.argtypes = [vp, vp, i64, i32, i32, i64, u64, vp, C.POINTER(_Plan), i32, C.c_double, i32,
                                          C.POINTER(_HostStats)]
        L.qrm_detect_host_multi.argtypes = [C.POINTER(vp), i32, vp, i64, i32, i32, i64, u64, vp, C.POINTER(_Plan), i32,
                                            C.POINTER(_HostStats)]
        L.qrm_extract_tiles_device.argtypes = [vp, vp, i64, i32, i32, i64, u64, i32, vp, vp]
        L.qrm_attack_device.argtypes = [vp, i64, i32, i32, i64, i32, C.c_double, vp, i64, C.POINTER(i32),
                                        C.POINTER(i32), vp]
        L.qrm_ppm_read.argtypes = [C.c_char_p, vp, i64, C.POINTER(i32), C.POINTER(i32)]
        L.qrm_ppm_write.argtypes = [C.c_char_p, vp, i32, i32]
        L.qrm_ppm_read_batch.argtypes = [C.POINTER(C.c_char_p), i64, i32, i32, vp, i64, i32, vp]
        L.qrm_records_json.argtypes = [vp, i64, i32, i32, i64, i32, i64, u64, vp, i64, C.POINTER(i64)]
        L.qrm_detect_device.argtypes = [vp, vp, i64, i32, i32, i64, u64, vp, vp]
        L.qrm_detect_host.argtypes = [vp, vp, i64, i32, i32, i64, u64, vp, C.POINTER(_Plan), i32,
                                      C.POINTER(_HostStats)]
        L.qrm_detect_ragged.argtypes = [vp, C.POINTER(vp), C.POINTER(i32), C.POINTER(i32), i64, u64, vp]
        L.qrm_extract_device.argtypes = [vp, vp, i64, i32, i32, i64, u64, vp, vp, vp]
        L.qrm_preprocess_host.argtypes = [vp, i32, i32, vp]
        L.qrm_rs_decode_packed_device.argtypes = [i32, i32, i32, vp, i64, vp, vp, i32, vp]
        L.qrm_rs_decode_symbols_device.argtypes = [i32, i32, i32, vp, i64, vp, vp, vp]
        L.qrm_rs_stress_device.argtypes = [i32, i32, i32, u64, i64, vp, vp, vp, vp]
        L.qrm_rs_stress_symbols_device.argtypes = [i32, i32, i32, u64, i64, vp, vp, vp, vp]
        L.qrm_rs_codebook_clear.argtypes = [i32, i32, i32, vp]
        L.qrm_warmup_saturation.argtypes = [vp, vp, i64, i32, i32, i64, i32, i32, vp, vp, vp]
        L.qrm_allocate_streams_sat.argtypes = [i32, vp, vp, vp, C.c_double, i32, i32, C.c_double, C.c_double, i32, vp, vp, C.POINTER(C.c_double)]
        L.qrm_device_cpus.argtypes = [i32, vp, i32, C.POINTER(i32)]
        L.qrm_rs_encode_packed.argtypes = [i32, i32, i32, u64, C.POINTER(u64)]
        L.qrm_verify_threshold.argtypes = [i32, C.c_double, C.POINTER(i32)]
        L.qrm_make_corpus_device.argtypes = [C.POINTER(_Config), u64, i64, i32, i32, i32, vp, vp]
        L.qrm_patterns_device.argtypes = [u64, i32, i32, vp, vp]
        L.qrm_allocate_streams.argtypes = [i32, vp, vp, C.c_double, i32, i32, C.c_double, C.c_double, i32, vp, vp,
                                           C.POINTER(C.c_double)]
        L.qrm_lpt_schedule.argtypes = [i32, vp, vp, vp, vp, i32, C.c_double, C.c_double, i32, i32, i32, vp, vp, vp,
                                       vp, vp, vp, C.POINTER(i32), vp, C.POINTER(i32)]
        L.qrm_warmup_profile.argtypes = [vp, vp, i64, i32, i32, i64, i32, i32, vp, vp]
        L.qrm_warmup_profile_mode.argtypes = [vp, vp, i64, i32, i32, i64, i32, i32, i32, vp, vp]
        L.qrm_ctx_set_plan.argtypes = [vp, C.POINTER(_Plan)]
        L.qrm_probe_decode_kernel.argtypes = [vp, vp, i64, i32, i32, i64, i32, C.POINTER(C.c_double)]
        L.qrm_hidden_detect_device.argtypes = [vp, vp, i64, i32, i32, i64, u64, u64, vp, vp, vp]
        L.qrm_resample_host.argtypes = [vp, i32, i32, i32, i32, i32, i32, i32, i32, i32, i32, vp]
        L.qrm_extract_float_host.argtypes = [u64, i32, i32, vp, vp]
        _lib = L
    return _lib


def _check(status: int):
    if status:
        raise _STATUS.get(status, QrmError)(lib().qrm_last_error().decode())


def _ptr(x) -> int:
    """Device/host address of a torch tensor or numpy array."""
    if hasattr(x, "data_ptr"):
        return x.data_ptr()
    if isinstance(x, np.ndarray):
        return x.ctypes.data
    if x is None:
        return 0
    return int(x)


_RAW_STREAM = None  # (torch._C._cuda_getCurrentRawStream, torch._C._cuda_getDevice) once CUDA is up


def _stream(stream=None) -> int:
    """CUDA stream handle: the given stream, else torch's current stream.

    The current stream is read through torch's raw accessors (0.2 us) rather
    than torch.cuda.current_stream() (3-4 us): per-call host cost bounds the
    back-to-back device-resident loop (bench.py's value)."""
    global _RAW_STREAM
    if stream is not None:
        return int(getattr(stream, "cuda_stream", stream))
    if _RAW_STREAM is not None:
        return _RAW_STREAM[0](_RAW_STREAM[1]())
    try:
        import torch
        if torch.cuda.is_available():
            s = torch.cuda.current_stream().cuda_stream
            get_raw = getattr(torch._C, "_cuda_getCurrentRawStream", None)
            get_dev = getattr(torch._C, "_cuda_getDevice", None)
            if get_raw is not None and get_dev is not None and get_raw(get_dev()) == s:
                _RAW_STREAM = (get_raw, get_dev)
            return s
    except ImportError:  # pragma: no cover
        pass
    return 0


def kernel_launch_count() -> int:
    return int(lib().qrm_kernel_launch_count())


# --------------------------------------------------------------- code / RS --
@dataclass(frozen=True)
class CodeParams:
    """CodeParams (rs.hpp:26-37): GF(2^m), (n, k), t = (n-k)//2, X_i = alpha^i."""
    m: int
    n: int
    k: int

    @property
    def t(self) -> int:
        return (self.n - self.k) // 2

    def message_bits(self) -> int:
        return self.k * self.m

    def codeword_bits(self) -> int:
        return self.n * self.m

    @staticmethod
    def make(m: int, n: int, k: int) -> "CodeParams":
        if m not in (4, 8):
            raise InvalidInput("symbol size must be 4 or 8")
        if n > (1 << m) - 1:
            raise InvalidInput("codeword length exceeds field bound")
        if k <= 0 or k >= n:
            raise InvalidInput("message length must satisfy 0 < k < n")
        return CodeParams(m, n, k)


def resolve_profile(name: str, payload_bits: int = 48) -> CodeParams:
    """resolve_profile (rs.cpp:65-76)."""
    if name == "gf16-15-12":
        return CodeParams.make(4, 15, 12)
    if name == "gf256-dynamic":
        if payload_bits <= 0 or payload_bits % 8:
            raise InvalidInput("gf256-dynamic payload must be a positive multiple of 8 bits")
        return CodeParams.make(8, payload_bits // 8 + 2, payload_bits // 8)
    raise InvalidInput(f"unknown code profile: {name}")


def bits_to_word(bits) -> int:
    w = 0
    for b in bits:
        w = (w << 1) | (int(b) & 1)
    return w


def word_to_bits(w: int, n: int) -> np.ndarray:
    return np.array([(int(w) >> (n - 1 - i)) & 1 for i in range(n)], dtype=np.uint8)


def default_message(key_seed: int, n_bits: int) -> np.ndarray:
    """default_message (cli.cpp:47-51): bit i = rng_word(key_seed, 0x6d73, i) & 1."""
    return np.array([rng_word(key_seed, 0x6D73, i) & 1 for i in range(n_bits)], dtype=np.uint8)


_M64 = (1 << 64) - 1


def mix64(x: int) -> int:
    """rng.hpp:15-22."""
    x ^= x >> 30
    x = (x * 0xBF58476D1CE4E5B9) & _M64
    x ^= x >> 27
    x = (x * 0x94D049BB133111EB) & _M64
    return x ^ (x >> 31)


def rng_word(seed: int, stream: int, ctr: int) -> int:
    """rng.hpp:25-28."""
    key = mix64((seed + 0x9E3779B97F4A7C15 * (stream + 1)) & _M64)
    return mix64(key ^ ((ctr * 0xD6E8FEB86659FD93) & _M64) ^ (ctr >> 32))


def rs_encode_packed(code: CodeParams, message: int) -> int:
    """rs_encode (rs.cpp:78-91) on a packed message."""
    out = C.c_uint64()
    _check(lib().qrm_rs_encode_packed(code.m, code.n, code.k, message, C.byref(out)))
    return out.value


def rs_stress_words(code: CodeParams, seed: int, count: int, device="cuda"):
    """Device RS stress words -> (msg, received, injected error count) torch tensors."""
    import torch
    msg = torch.empty(count, dtype=torch.int64, device=device)
    words = torch.empty(count, dtype=torch.int64, device=device)
    ne = torch.empty(count, dtype=torch.int8, device=device)
    _check(lib().qrm_rs_stress_device(code.m, code.n, code.k, seed, count, _ptr(msg), _ptr(words), _ptr(ne),
                                      _stream()))
    return msg, words, ne


def rs_stress_symbols(code: CodeParams, seed: int, count: int, device="cuda"):
    """Device RS stress words of a symbol code -> (true codewords, received words, injected
    error count): uint8 [count, n], uint8 [count, n], int8 [count]."""
    import torch
    true_cw = torch.empty((count, code.n), dtype=torch.uint8, device=device)
    recv = torch.empty((count, code.n), dtype=torch.uint8, device=device)
    ne = torch.empty(count, dtype=torch.int8, device=device)
    _check(lib().qrm_rs_stress_symbols_device(code.m, code.n, code.k, seed, count, _ptr(true_cw), _ptr(recv),
                                              _ptr(ne), _stream()))
    return true_cw, recv, ne


def bw_decode_symbols_into(code: CodeParams, recv, cw_out, nerr_out, stream=None):
    """bw_decode_symbols writing into caller tensors (timed loops)."""
    _check(lib().qrm_rs_decode_symbols_device(code.m, code.n, code.k, _ptr(recv), recv.shape[0], _ptr(cw_out),
                                              _ptr(nerr_out), _stream(stream)))
    return cw_out, nerr_out


def rs_codebook_clear(code: CodeParams, stream=None):
    """Empty the device codebook (algo 3 of bw_decode_packed) for `code`."""
    _check(lib().qrm_rs_codebook_clear(code.m, code.n, code.k, _stream(stream)))


def bw_decode_packed(code: CodeParams, words, cw_out=None, nerr_out=None, algo: int = 0, stream=None):
    """Batched bw_decode (rs.cpp:188-196) on the GPU, packed words (n*m <= 64).

    ``words`` is a CUDA int64 tensor; returns (codewords, errors_corrected or -1)."""
    import torch
    count = words.numel()
    if cw_out is None:
        cw_out = torch.empty_like(words)
    if nerr_out is None:
        nerr_out = torch.empty(count, dtype=torch.int8, device=words.device)
    _check(lib().qrm_rs_decode_packed_device(code.m, code.n, code.k, _ptr(words), count, _ptr(cw_out),
                                             _ptr(nerr_out), algo, _stream(stream)))
    return cw_out, nerr_out


def bw_decode_symbols(code: CodeParams, recv, stream=None):
    """Batched bw_decode on symbol rows (uint8 CUDA tensor [count, n]); warp-per-codeword BM."""
    import torch
    count = recv.shape[0]
    cw = torch.empty_like(recv)
    ne = torch.empty(count, dtype=torch.int8, device=recv.device)
    _check(lib().qrm_rs_decode_symbols_device(code.m, code.n, code.k, _ptr(recv), count, _ptr(cw), _ptr(ne),
                                              _stream(stream)))
    return cw, ne


def bw_decode(bits, code: CodeParams):
    """Single-word bw_decode (rs.hpp:57) -> (message bits, codeword bits, errors) or None.

    Runs on the GPU (a batch of one); prefer the batched calls."""
    import torch
    bits = np.asarray(bits, dtype=np.uint8)
    if bits.size != code.codeword_bits():
        raise InvalidInput("received bit length does not match profile")
    if code.codeword_bits() <= 64:
        w = torch.tensor([np.int64(np.uint64(bits_to_word(bits)).view(np.int64))], device="cuda")
        cw, ne = bw_decode_packed(code, w)
        e = int(ne.item())
        if e < 0:
            return None
        cwb = word_to_bits(int(cw.item()) & _M64, code.codeword_bits())
    else:
        sym = bits.reshape(code.n, code.m)
        vals = (sym * (1 << np.arange(code.m - 1, -1, -1))).sum(1).astype(np.uint8)
        cw, ne = bw_decode_symbols(code, torch.tensor(vals, device="cuda").view(1, -1))
        e = int(ne.item())
        if e < 0:
            return None
        s = cw.cpu().numpy()[0]
        cwb = np.array([(int(v) >> (code.m - 1 - b)) & 1 for v in s for b in range(code.m)], np.uint8)
    return cwb[: code.message_bits()].copy(), cwb, e


def verify_threshold(n_bits: int, fpr: float) -> int:
    """verify_threshold (detect.cpp:31-66)."""
    t = C.c_int()
    _check(lib().qrm_verify_threshold(n_bits, fpr, C.byref(t)))
    return t.value


# ------------------------------------------------------------- detection --
@dataclass
class DetectionConfig:
    """DetectionConfig (detect.hpp:25-37) with the reference defaults (cli.cpp:55-65)."""
    profile: str = "gf16-15-12"
    payload_bits: int = 48
    tile_size: int = 64
    tile_strategy: str = "random_grid"
    tile_seed: int = 0
    key_seed: int = 1
    alpha: float = 0.04
    fpr_target: float = 1e-6
    key_message: np.ndarray | None = None
    code: CodeParams | None = field(default=None)
    # extractor behind the WatermarkCodec plug-in point: "spread_spectrum" (the
    # reference's SpreadSpectrumCodec) or "conv" (learned conv stack, weights
    # drawn from conv_seed; oracle/hidden_oracle.c is its contract)
    extractor: str = "spread_spectrum"
    conv_seed: int = 7

    def __post_init__(self):
        if self.code is None:
            self.code = resolve_profile(self.profile, self.payload_bits)
        if self.key_message is None:
            self.key_message = default_message(self.key_seed, self.code.message_bits())
        self.key_message = np.ascontiguousarray(self.key_message, dtype=np.uint8)

    def _c(self) -> _Config:
        if self.tile_strategy not in TILE_STRATEGY:
            raise InvalidInput(f"unknown tile strategy: {self.tile_strategy}")
        return _Config(self.code.m, self.code.n, self.code.k, self.tile_size, TILE_STRATEGY[self.tile_strategy],
                       self.tile_seed, self.key_seed, self.alpha,
                       self.key_message.ctypes.data_as(C.POINTER(C.c_uint8)), self.fpr_target)


def make_corpus(cfg: DetectionConfig, first_seed: int, count: int, w: int = 256, h: int = 256, embed: bool = True,
                out=None, stream=None):
    """Synthetic corpus on the device (cmd_bench recipe, cli.cpp:404-411) -> uint8 CUDA tensor [count, h, w, 3]."""
    import torch
    if out is None:
        out = torch.empty((count, h, w, 3), dtype=torch.uint8, device="cuda")
    c = cfg._c()
    _check(lib().qrm_make_corpus_device(C.byref(c), first_seed, count, w, h, int(embed), _ptr(out), _stream(stream)))
    return out


def patterns(key_seed: int, n_bits: int, l: int):
    """The codec's +-1 planes (stego.cpp:22-26) as an int8 CUDA tensor [n_bits, 3 l^2]."""
    import torch
    out = torch.empty((n_bits, 3 * l * l), dtype=torch.int8, device="cuda")
    _check(lib().qrm_patterns_device(key_seed, n_bits, l, _ptr(out), _stream()))
    return out


def preprocess(img: np.ndarray) -> np.ndarray:
    """preprocess (transforms.cpp:42-47) on the GPU: u8 HxWx3 -> float32 256x256x3."""
    im = np.ascontiguousarray(img, dtype=np.uint8)
    out = np.zeros((256, 256, 3), np.float32)
    _check(lib().qrm_preprocess_host(im.ctypes.data, im.shape[1], im.shape[0], out.ctypes.data))
    return out


_U8 = None  # torch.uint8, bound on first use (torch is imported lazily)


def _device_images(images, device: int):
    """Check a device image batch before its address crosses the C-ABI: uint8
    CUDA tensor [B, H, W, 3] on the context's GPU whose rows and pixels are
    contiguous (any batch stride). Other layouts are made contiguous; a CPU
    tensor or one on another GPU is an error (no silent fallback). The common
    case costs ~1 us (bench.py's back-to-back loop is sensitive to host time)."""
    global _U8
    if _U8 is None:
        import torch
        _U8 = torch.uint8
    try:
        ok = images.dtype == _U8 and images.is_cuda and images.get_device() == device and images.dim() == 4
    except AttributeError:
        raise InvalidInput("images must be a CUDA torch.Tensor") from None
    if not ok:
        if images.dtype != _U8:
            raise InvalidInput(f"images must be uint8, got {images.dtype}")
        if not images.is_cuda:
            raise InvalidInput("images must be on a CUDA device (use detect_host for host images)")
        if images.get_device() != device:
            raise InvalidInput(f"images are on cuda:{images.get_device()}, the context on cuda:{device}")
        raise InvalidInput(f"images must be [B, H, W, 3] (interleaved RGB), got {tuple(images.shape)}")
    if images.shape[3] != 3:
        raise InvalidInput(f"images must be [B, H, W, 3] (interleaved RGB), got {tuple(images.shape)}")
    if not images.is_contiguous():
        B, H, W, _ = images.shape
        st = images.stride()
        if B > 0 and (st[3] != 1 or st[2] != 3 or st[1] != 3 * W or (B > 1 and st[0] < H * W * 3)):
            images = images.contiguous()
    return images


class DetectionContext:
    """DetectionContext (detect.hpp:101-119): codec patterns, key codeword, thresholds on one GPU."""

    def __init__(self, cfg: DetectionConfig, device: int = 0):
        self.cfg = cfg
        self.device = device
        h = C.c_void_p()
        c = cfg._c()
        if cfg.extractor not in EXTRACTOR:
            raise InvalidInput(f"unknown extractor: {cfg.extractor}")
        _check(lib().qrm_ctx_create(device, C.byref(c), C.byref(h)))
        self._h = h
        if EXTRACTOR[cfg.extractor]:
            _check(lib().qrm_ctx_set_extractor(h, EXTRACTOR[cfg.extractor], cfg.conv_seed))  # close() frees h
        cw, msg, tm, tr = C.c_uint64(), C.c_uint64(), C.c_int(), C.c_int()
        _check(lib().qrm_ctx_info(h, C.byref(cw), C.byref(msg), C.byref(tm), C.byref(tr)))
        self.key_codeword, self.key_message, self.tau_message, self.tau_raw = cw.value, msg.value, tm.value, tr.value

    @property
    def window_bytes(self) -> int:
        """Algorithmic bytes read per image: the l x l x 3 u8 tile window."""
        return 3 * self.cfg.tile_size * self.cfg.tile_size

    def kernel_time_probe(self, images, reps: int = 20) -> float:
        """Mean duration (ms) of the decode kernel alone on a device batch."""
        images = _device_images(images, self.device)
        B, H, W, _ = images.shape
        ms = C.c_double()
        _check(lib().qrm_probe_decode_kernel(self._h, _ptr(images), B, W, H, images.stride(0), reps, C.byref(ms)))
        return ms.value

    def close(self):
        if getattr(self, "_h", None):
            lib().qrm_ctx_destroy(self._h)
            self._h = None

    def __del__(self):  # pragma: no cover
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    def detect_device(self, images, first_draw: int = 0, out=None, stream=None):
        """Device-resident batch: images uint8 CUDA tensor [B, H, W, 3] -> record tensor [B, 24] (uint8)."""
        images = _device_images(images, self.device)
        B, H, W, _ = images.shape
        if out is None:
            import torch
            out = torch.empty((B, RECORD_DTYPE.itemsize), dtype=torch.uint8, device=images.device)
        _check(lib().qrm_detect_device(self._h, _ptr(images), B, W, H, images.stride(0), first_draw, _ptr(out),
                                       _stream(stream)))
        return out

    def hidden_detect_device(self, images, weight_seed: int = 7, first_draw: int = 0, logits: bool = True,
                             out=None, stream=None):
        """Learned extractor (HiDDeN-style conv stack on tcgen05, bf16) + RS + verify on a device batch.

        -> (logits float32 [B, N] or None, record tensor [B, 24] uint8)."""
        import torch
        images = _device_images(images, self.device)
        B, H, W, _ = images.shape
        nb = self.cfg.code.codeword_bits()
        lg = torch.empty((B, nb), dtype=torch.float32, device=images.device) if logits else None
        if out is None:
            out = torch.empty((B, RECORD_DTYPE.itemsize), dtype=torch.uint8, device=images.device)
        _check(lib().qrm_hidden_detect_device(self._h, _ptr(images), B, W, H, images.stride(0), first_draw,
                                              weight_seed, _ptr(lg), _ptr(out), _stream(stream)))
        return lg, out

    def extract_tiles(self, images, first_draw: int = 0, channels: int = 3, out=None, stream=None):
        """preprocess -> select_tile -> extract_tile -> normalize as bf16 NHWC tiles
        [B, l, l, channels] on the device (channels 4: zero-padded)."""
        import torch
        images = _device_images(images, self.device)
        B, H, W, _ = images.shape
        l = self.cfg.tile_size
        if out is None:
            out = torch.empty((B, l, l, channels), dtype=torch.bfloat16, device=images.device)
        _check(lib().qrm_extract_tiles_device(self._h, _ptr(images), B, W, H, images.stride(0), first_draw, channels,
                                              _ptr(out), _stream(stream)))
        return out

    def extract_device(self, images, first_draw: int = 0, soft: bool = True, stream=None):
        """SpreadSpectrumCodec::extract + harden on a device batch -> (soft float64 [B, N] or None, raw int64 [B])."""
        images = _device_images(images, self.device)
        import torch
        B, H, W, _ = images.shape
        nb = self.cfg.code.codeword_bits()
        s = torch.empty((B, nb), dtype=torch.float64, device=images.device) if soft else None
        raw = torch.empty(B, dtype=torch.int64, device=images.device)
        _check(lib().qrm_extract_device(self._h, _ptr(images), B, W, H, images.stride(0), first_draw, _ptr(s),
                                        _ptr(raw), _stream(stream)))
        return s, raw

    def detect_host(self, images: np.ndarray | None = None, first_draw: int = 0, plan=None, mode: int = 0,
                    out: np.ndarray | None = None, ptr: int | None = None, shape=None, lpt=None):
        """Host images (pinned or pageable) -> host records, through the stream executor.

        ``images``: numpy uint8 [B, H, W, 3] (or pass ``ptr``+``shape`` for a pinned torch buffer).
        ``mode``: transfer stage -- 0 zero-copy window fetch, 1 full-image H2D, 2 host-staged
        windows, 3 both 0 and 2 on each mini-batch (see set_transfer_split).
        Returns (records structured array, stats dict)."""
        if images is not None:
            images = np.ascontiguousarray(images, dtype=np.uint8)
            B, H, W, _ = images.shape
            p = images.ctypes.data
            stride = H * W * 3
        else:
            B, H, W = shape
            p = ptr
            stride = H * W * 3
        if out is None:
            out = np.zeros(B, dtype=RECORD_DTYPE)
        st = _HostStats()
        pl = None
        if plan is not None:
            pl = _Plan((C.c_int * 3)(*plan[0]), (C.c_int * 3)(*plan[1]))
        if lpt is not None:  # (lambda, b_min): Algorithm 2 assigns the mini-batches to decode streams
            _check(lib().qrm_detect_host_lpt(self._h, p, B, W, H, stride, first_draw, out.ctypes.data,
                                             C.byref(pl) if pl is not None else None, mode, float(lpt[0]),
                                             int(lpt[1]), C.byref(st)))
        else:
            _check(lib().qrm_detect_host(self._h, p, B, W, H, stride, first_draw, out.ctypes.data,
                                         C.byref(pl) if pl is not None else None, mode, C.byref(st)))
        return out, {"wall_ms": st.wall_ms, "h2d_bytes": st.h2d_bytes, "d2h_bytes": st.d2h_bytes,
                     "minibatches": st.minibatches, "kernel_launches": st.kernel_launches}

    def detect_images(self, images, first_draw: int = 0, plan=None, load=None, image_ns: bool = False):
        """detect_batch over separate same-size host images (a list of HxWx3 uint8
        arrays, >= 256 px): only each image's window is gathered into the context's
        pinned staging ring and copied. ``load``: SyntheticStageLoad ns per image
        (transfer, decode, correct). Returns (records, {"wall_ns", "busy_ns",
        "image_ns" [B, 3] when asked})."""
        keep = [np.ascontiguousarray(im, dtype=np.uint8) for im in images]
        n = len(keep)
        if n == 0:
            return np.zeros(0, dtype=RECORD_DTYPE), {"wall_ns": 0, "busy_ns": [0, 0, 0]}
        H, W = keep[0].shape[:2]
        ptrs = (C.c_void_p * n)(*[a.ctypes.data for a in keep])
        out = np.zeros(n, dtype=RECORD_DTYPE)
        pl = _Plan((C.c_int * 3)(*plan[0]), (C.c_int * 3)(*plan[1])) if plan is not None else None
        ld = _StageLoad((C.c_int64 * 3)(*(load or (0, 0, 0))))
        ins = np.zeros((n, 3), np.int64) if image_ns else None
        tm = _StageTimes(0, (C.c_int64 * 3)(0, 0, 0), ins.ctypes.data if ins is not None else None)
        _check(lib().qrm_detect_host_images(self._h, ptrs, n, W, H, first_draw, out.ctypes.data,
                                            C.byref(pl) if pl is not None else None, C.byref(ld), C.byref(tm)))
        info = {"wall_ns": tm.wall_ns, "busy_ns": list(tm.busy_ns)}
        if ins is not None:
            info["image_ns"] = ins
        return out, info

    def detect_host_timed(self, images: np.ndarray, first_draw: int = 0, plan=None, mode: int = 0, load=None):
        """qrm_detect_host with SyntheticStageLoad and DeskReport-style stage spans
        -> (records, {"wall_ns", "busy_ns", "image_ns" [B, 3]})."""
        images = np.ascontiguousarray(images, dtype=np.uint8)
        B, H, W, _ = images.shape
        out = np.zeros(B, dtype=RECORD_DTYPE)
        pl = _Plan((C.c_int * 3)(*plan[0]), (C.c_int * 3)(*plan[1])) if plan is not None else None
        ld = _StageLoad((C.c_int64 * 3)(*(load or (0, 0, 0))))
        ins = np.zeros((B, 3), np.int64)
        tm = _StageTimes(0, (C.c_int64 * 3)(0, 0, 0), ins.ctypes.data)
        _check(lib().qrm_detect_host_timed(self._h, images.ctypes.data, B, W, H, H * W * 3, first_draw,
                                           out.ctypes.data, C.byref(pl) if pl is not None else None, mode,
                                           C.byref(ld), C.byref(tm)))
        return out, {"wall_ns": tm.wall_ns, "busy_ns": list(tm.busy_ns), "image_ns": ins}

    def detect_ragged(self, images, first_draw: int = 0) -> np.ndarray:
        """Mixed-size host images (list of HxWx3 uint8) -> records."""
        keep = [np.ascontiguousarray(im, dtype=np.uint8) for im in images]
        n = len(keep)
        ptrs = (C.c_void_p * n)(*[a.ctypes.data for a in keep])
        ws = (C.c_int * n)(*[a.shape[1] for a in keep])
        hs = (C.c_int * n)(*[a.shape[0] for a in keep])
        out = np.zeros(n, dtype=RECORD_DTYPE)
        _check(lib().qrm_detect_ragged(self._h, ptrs, ws, hs, n, first_draw, out.ctypes.data))
        return out

    def set_input_overlap(self, enable: bool):
        """qrm_ctx_set_input_overlap: promise that detect_device's images are complete
        before the preceding kernel on the stream (resident batches decoded back to
        back), letting each decode's window loads overlap the previous decode."""
        _check(lib().qrm_ctx_set_input_overlap(self._h, int(bool(enable))))

    def set_transfer_split(self, zero_copy_fraction: float):
        """Host pipeline mode 3: share of each mini-batch's windows fetched zero-copy."""
        _check(lib().qrm_ctx_set_transfer_split(self._h, float(zero_copy_fraction)))

    def set_plan(self, streams, minibatch):
        pl = _Plan((C.c_int * 3)(*streams), (C.c_int * 3)(*minibatch))
        _check(lib().qrm_ctx_set_plan(self._h, C.byref(pl)))

    def warmup_profile(self, images: np.ndarray | None = None, iters: int = 3, b0: int = 16, mode: int = 1,
                       ptr: int | None = None, shape=None):
        """warmup_profile (sim.cpp:240-288) on the device stages -> (time[3] ms per b0, memory[3] B/image).
        mode: the host pipeline's transfer (0 window fetch, 1 full-image copy)."""
        if images is not None:
            images = np.ascontiguousarray(images, dtype=np.uint8)
            B, H, W, _ = images.shape
            p = images.ctypes.data
        else:
            B, H, W = shape
            p = ptr
        t = np.zeros(3)
        m = np.zeros(3)
        _check(lib().qrm_warmup_profile_mode(self._h, p, B, W, H, H * W * 3, iters, b0, mode, t.ctypes.data,
                                             m.ctypes.data))
        return t, m

    def warmup_saturation(self, images: np.ndarray | None = None, iters: int = 3, b0: int = 512,
                          ptr: int | None = None, shape=None):
        """GPU-aware warm-up (extension): the mode-0 stages on 1, 2 and 4 concurrent
        streams -> (time[3] ms per b0 on one stream, memory[3] B/image, sat[3] best speedup)."""
        if images is not None:
            images = np.ascontiguousarray(images, dtype=np.uint8)
            B, H, W, _ = images.shape
            p = images.ctypes.data
        else:
            B, H, W = shape
            p = ptr
        t, m, sat = np.zeros(3), np.zeros(3), np.zeros(3)
        _check(lib().qrm_warmup_saturation(self._h, p, B, W, H, H * W * 3, iters, b0, t.ctypes.data,
                                           m.ctypes.data, sat.ctypes.data))
        return t, m, sat


def device_cpus(device: int) -> list:
    """Host CPUs on GPU `device`'s NUMA node ([] when unknown)."""
    n = C.c_int32()
    buf = np.zeros(4096, np.int32)
    _check(lib().qrm_device_cpus(device, buf.ctypes.data, buf.size, C.byref(n)))
    return buf[:min(n.value, buf.size)].tolist()


def pin_to_device(device: int) -> list:
    """Pin this process to GPU `device`'s NUMA-local CPUs (before allocating pinned
    host buffers, so first touch lands on that node). Returns the CPU list used."""
    cpus = device_cpus(device)
    usable = sorted(set(cpus) & os.sched_getaffinity(0)) if cpus else []
    if usable:
        os.sched_setaffinity(0, usable)
    return usable

def detect_host_multi(contexts, images: np.ndarray, first_draw: int = 0, plan=None, mode: int = 0, out=None):
    """qrm_detect_host_multi: one contiguous shard per context (normally one per GPU),
    each on its own host thread, records at their global positions -> (records, stats)."""
    images = np.ascontiguousarray(images, dtype=np.uint8)
    B, H, W, _ = images.shape
    if out is None:
        out = np.zeros(B, dtype=RECORD_DTYPE)
    hs = (C.c_void_p * len(contexts))(*[c._h.value if hasattr(c._h, "value") else c._h for c in contexts])
    st = _HostStats()
    pl = _Plan((C.c_int * 3)(*plan[0]), (C.c_int * 3)(*plan[1])) if plan is not None else None
    _check(lib().qrm_detect_host_multi(hs, len(contexts), images.ctypes.data, B, W, H, H * W * 3, first_draw,
                                       out.ctypes.data, C.byref(pl) if pl is not None else None, mode, C.byref(st)))
    return out, {"wall_ms": st.wall_ms, "h2d_bytes": st.h2d_bytes, "d2h_bytes": st.d2h_bytes,
                 "minibatches": st.minibatches, "kernel_launches": st.kernel_launches}


def records_from_device(t) -> np.ndarray:
    """uint8 record tensor [B, 24] -> structured numpy array."""
    return np.ascontiguousarray(t.cpu().numpy()).view(RECORD_DTYPE).reshape(-1)


def detect_batch(images, cfg: DetectionConfig, plan=None, first_draw: int = 0, device: int = 0, mode: int = 0):
    """detect_batch (detect.cpp:250): list/array of host images -> records (structured array).

    A uniform uint8 array goes through the stream executor (``mode``); a list of
    same-size images of >= 256 px through the per-image staged path; mixed sizes
    through the ragged path."""
    with DetectionContext(cfg, device) as ctx:
        if isinstance(images, np.ndarray) and images.ndim == 4:
            return ctx.detect_host(images, first_draw, plan=plan, mode=mode)[0]
        images = list(images)
        if images and all(np.shape(im) == np.shape(images[0]) for im in images) and min(np.shape(images[0])[:2]) >= 256:
            return ctx.detect_images(images, first_draw, plan=plan)[0]
        return ctx.detect_ragged(images, first_draw)


def semantic_fields(rec: np.ndarray, code: CodeParams) -> dict:
    """Record fields compared by semantic_equal (detect.cpp:25-29)."""
    nb = code.codeword_bits()
    return {"raw": rec["raw"].astype(np.uint64), "decoded": rec["status"] == 1,
            "msg": np.where(rec["status"] == 1, rec["msg"], 0).astype(np.uint64),
            "errors": rec["errors"].astype(np.int32), "bit_acc": rec["matches"] / float(nb),
            "verified": rec["verified"].astype(bool)}


ATTACKS = ("centercrop", "resizeto", "normalize", "crop", "resize", "brightness", "contrast", "saturation",
           "sharpness", "blur", "overlay_text", "jpeg_approx")  # TransformOp order (transforms.hpp:22-35)
ATTACK_SUITE = (("C-0.1", "crop", 0.1), ("C-0.5", "crop", 0.5), ("R-0.5", "resize", 0.5), ("BL", "blur", 1.0),
                ("BR-2", "brightness", 2.0), ("CON-2", "contrast", 2.0))  # attack_suite (transforms.cpp:364-373)


def apply_attack(images, op: str, param: float, stream=None):
    """apply_attack (transforms.cpp:289-362) on a uint8 CUDA tensor [B, H, W, 3] -> CUDA tensor
    (uint8, or float32 for "normalize"), bit-exact with the reference."""
    import torch
    if op not in ATTACKS:
        raise InvalidInput(f"unknown transform op: {op}")
    B, H, W, _ = images.shape
    code = ATTACKS.index(op)
    ow, oh = C.c_int(), C.c_int()
    _check(lib().qrm_attack_device(_ptr(images), B, W, H, images.stride(0), code, param, None, 0, C.byref(ow),
                                   C.byref(oh), _stream(stream)))
    dt = torch.float32 if op == "normalize" else torch.uint8
    out = torch.empty((B, oh.value, ow.value, 3), dtype=dt, device=images.device)
    _check(lib().qrm_attack_device(_ptr(images), B, W, H, images.stride(0), code, param, _ptr(out),
                                   out.stride(0) * out.element_size(), C.byref(ow), C.byref(oh), _stream(stream)))
    return out


# --------------------------------------------------------------- formats --
def read_ppm(path) -> np.ndarray:
    """read_ppm (image.cpp:129-146) -> uint8 [H, W, 3]."""
    w, h = C.c_int(), C.c_int()
    p = os.fsencode(path)
    _check(lib().qrm_ppm_read(p, None, 0, C.byref(w), C.byref(h)))
    out = np.empty((h.value, w.value, 3), np.uint8)
    _check(lib().qrm_ppm_read(p, out.ctypes.data, out.nbytes, C.byref(w), C.byref(h)))
    return out


def write_ppm(img: np.ndarray, path) -> None:
    """write_ppm (image.cpp:148-156)."""
    img = np.ascontiguousarray(img, np.uint8)
    _check(lib().qrm_ppm_write(os.fsencode(path), img.ctypes.data, img.shape[1], img.shape[0]))


def read_ppm_batch(paths, out=None, threads: int = 0):
    """ingest (cli.cpp:22-45) of same-size P6 files, decoded in parallel straight
    into `out` (uint8 [N, H, W, 3]; numpy or a pinned torch tensor)."""
    paths = [os.fsencode(p) for p in paths]
    w, h = C.c_int(), C.c_int()
    _check(lib().qrm_ppm_read(paths[0], None, 0, C.byref(w), C.byref(h)))
    if out is None:
        out = np.empty((len(paths), h.value, w.value, 3), np.uint8)
    arr = (C.c_char_p * len(paths))(*paths)
    _check(lib().qrm_ppm_read_batch(arr, len(paths), w.value, h.value, _ptr(out), h.value * w.value * 3,
                                    threads or (os.cpu_count() or 1), None))
    return out


def records_json(rec: np.ndarray, code: CodeParams, first_index: int = 0, cache=(True, 4096, 1 << 20)) -> str:
    """The "records" array of cmd_detect's report (cli.cpp:279-281), record_to_json
    (json_io.cpp:98-120) per record in nlohmann dump(2) layout; cache_hit from the
    CorrectionCache policy (enabled, capacity, stale_after) in index order."""
    rec = np.ascontiguousarray(rec)
    n = C.c_int64()
    nb, kb = code.codeword_bits(), code.message_bits()
    en, capy, stale = int(cache[0]), int(cache[1]), int(cache[2])
    _check(lib().qrm_records_json(rec.ctypes.data, len(rec), nb, kb, first_index, en, capy, stale, None, 0,
                                  C.byref(n)))
    buf = C.create_string_buffer(n.value + 1)
    _check(lib().qrm_records_json(rec.ctypes.data, len(rec), nb, kb, first_index, en, capy, stale, buf,
                                  n.value + 1, C.byref(n)))
    return buf.value.decode()


# ------------------------------------------------------------- scheduler --
@dataclass
class StreamPlan:
    """StreamPlan (sched.hpp:26-34)."""
    streams: list
    minibatch: list
    bottleneck: float = 0.0


def allocate_streams(time, memory, b0: float, global_batch: int, stream_budget: int, m_cap: float,
                     epsilon: float, stall_cap: int) -> StreamPlan:
    """allocate_streams (sched.cpp:50-114): the paper's Algorithm 1."""
    K = len(time)
    t = np.ascontiguousarray(time, np.float64)
    u = np.ascontiguousarray(memory, np.float64)
    s = np.zeros(K, np.int32)
    m = np.zeros(K, np.int32)
    bn = C.c_double()
    _check(lib().qrm_allocate_streams(K, t.ctypes.data, u.ctypes.data, b0, global_batch, stream_budget, m_cap,
                                      epsilon, stall_cap, s.ctypes.data, m.ctypes.data, C.byref(bn)))
    return StreamPlan(s.tolist(), m.tolist(), bn.value)


def allocate_streams_sat(time, memory, sat, b0: float, global_batch: int, stream_budget: int, m_cap: float,
                         epsilon: float, stall_cap: int) -> StreamPlan:
    """Algorithm 1 with the GPU-aware stage model (extension): stage k's speedup from
    s streams is capped at the measured sat[k]."""
    K = len(time)
    if len(sat) != K or len(memory) != K:
        raise InvalidInput("profile saturation length mismatch")
    t = np.ascontiguousarray(time, np.float64)
    u = np.ascontiguousarray(memory, np.float64)
    sa = np.ascontiguousarray(sat, np.float64)
    s = np.zeros(K, np.int32)
    m = np.zeros(K, np.int32)
    bn = C.c_double()
    _check(lib().qrm_allocate_streams_sat(K, t.ctypes.data, u.ctypes.data, sa.ctypes.data, b0, global_batch,
                                          stream_budget, m_cap, epsilon, stall_cap, s.ctypes.data, m.ctypes.data,
                                          C.byref(bn)))
    return StreamPlan(s.tolist(), m.tolist(), bn.value)

def lpt_schedule(ids, latency, memory, units, stream_count: int, lam: float, m_cap: float, b_min: int,
                 global_batch: int) -> dict:
    """lpt_schedule (sched.cpp:177-235): the paper's Algorithm 2.

    Returns {"pieces": [(stream, id, units, latency, memory, mb)], "loads": [...], "m_unit": int}."""
    n = len(ids)
    ids_ = np.ascontiguousarray(ids, np.int32)
    lat = np.ascontiguousarray(latency, np.float64)
    mem = np.ascontiguousarray(memory, np.float64)
    un = np.ascontiguousarray(units, np.int32)
    cap = int(un.sum()) + n + 1
    ps, pi, pu, pm = (np.zeros(cap, np.int32) for _ in range(4))
    pl, pme = np.zeros(cap), np.zeros(cap)
    npieces, mu = C.c_int(), C.c_int()
    loads = np.zeros(stream_count)
    _check(lib().qrm_lpt_schedule(n, ids_.ctypes.data, lat.ctypes.data, mem.ctypes.data, un.ctypes.data,
                                  stream_count, lam, m_cap, b_min, global_batch, cap, ps.ctypes.data, pi.ctypes.data,
                                  pu.ctypes.data, pl.ctypes.data, pme.ctypes.data, pm.ctypes.data, C.byref(npieces),
                                  loads.ctypes.data, C.byref(mu)))
    c = npieces.value
    return {"pieces": list(zip(ps[:c].tolist(), pi[:c].tolist(), pu[:c].tolist(), pl[:c].tolist(),
                               pme[:c].tolist(), pm[:c].tolist())), "loads": loads.tolist(), "m_unit": mu.value}
