"""The C-ABI library: loads, exports exactly what include/qrmark_gpu.h declares,
and its host-only entry points (planners, encoder, thresholds) match the
reference's golden vectors. CPU only — no compute call runs without a GPU."""
import json
import os
import re
import subprocess

import numpy as np
import pytest

import paper_2509_02447_b200 as q

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
G = os.path.join(ROOT, "tests", "golden")


def header_symbols():
    src = open(os.path.join(ROOT, "include", "qrmark_gpu.h")).read()
    return set(re.findall(r"QRM_EXPORT\s+[\w\s\*]+?\b(qrm_\w+)\s*\(", src))


def test_library_loads_and_exports_header():
    L = q.lib()
    assert L is not None
    declared = header_symbols()
    assert declared == set(q.ABI_SYMBOLS), declared ^ set(q.ABI_SYMBOLS)
    out = subprocess.run(["nm", "-D", "--defined-only", q.LIB_PATH], capture_output=True, text=True).stdout
    exported = {ln.split()[-1] for ln in out.splitlines() if " T qrm_" in ln}
    assert declared <= exported, declared - exported
    for s in declared:
        assert hasattr(L, s)


def test_library_is_sm100a():
    out = subprocess.run(["cuobjdump", "-lelf", q.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    sass = subprocess.run(["cuobjdump", "-sass", q.LIB_PATH], capture_output=True, text=True).stdout
    assert "UTCIMMA" in sass and "LDTM" in sass  # tcgen05.mma kind::i8 + tcgen05.ld


@pytest.fixture(scope="module")
def kat():
    with open(os.path.join(G, "kat.json")) as f:
        return json.load(f)


def test_host_thresholds_and_encoder(kat):
    for n, tau in kat["tau_1e-6"].items():
        assert q.verify_threshold(int(n), 1e-6) == tau
    for n, f, tau in kat["tau_misc"]:
        assert q.verify_threshold(n, f) == tau
    with pytest.raises(q.InvalidInput):
        q.verify_threshold(0, 1e-6)
    msg = int(kat["default_message_hex"], 16)
    assert q.rs_encode_packed(q.resolve_profile("gf16-15-12"), msg) == int(kat["gf16_codeword_hex"], 16)
    assert q.rs_encode_packed(q.resolve_profile("gf256-dynamic", 48), msg) == int(kat["gf256_codeword_hex"], 16)
    assert q.bits_to_word(q.default_message(1, 48)) == msg
    with pytest.raises(q.InvalidInput):
        q.resolve_profile("nope")
    with pytest.raises(q.InvalidInput):
        q.resolve_profile("gf256-dynamic", 42)


def test_planners_match_reference(kat):
    for c in kat["allocate_streams"]:
        if c["rc"] == 0:
            p = q.allocate_streams(c["time"], c["memory"], c["b0"], c["B"], c["P"], c["m_cap"], c["eps"], c["stall"])
            assert (p.streams, p.minibatch, p.bottleneck) == (c["streams"], c["minibatch"], c["bottleneck"])
        else:
            with pytest.raises((q.InvalidInput, q.InfeasibleConfig)):
                q.allocate_streams(c["time"], c["memory"], c["b0"], c["B"], c["P"], c["m_cap"], c["eps"],
                                   c["stall"])
    for c in kat["lpt_schedule"]:
        lam = float("inf") if c["lam"] == "inf" else c["lam"]
        if c["rc"] == 0:
            out = q.lpt_schedule(c["ids"], c["lat"], c["mem"], c["units"], c["S"], lam, c["m_cap"], c["b_min"],
                                 c["B"])
            assert [list(p) for p in out["pieces"]] == [list(p) for p in c["out"]["pieces"]]
            assert out["loads"] == c["out"]["loads"] and out["m_unit"] == c["out"]["m_unit"]
        else:
            with pytest.raises(q.InfeasibleConfig):
                q.lpt_schedule(c["ids"], c["lat"], c["mem"], c["units"], c["S"], lam, c["m_cap"], c["b_min"],
                               c["B"])


def test_gpu_aware_allocate_streams(kat):
    """The saturation-capped Algorithm 1 (extension) equals the reference's when no
    stage saturates below the stream budget, and never adds streams to a stage
    whose measured speedup is 1."""
    for c in kat["allocate_streams"]:
        if c["rc"] != 0:
            continue
        sat = [float(c["P"])] * len(c["time"])
        p = q.allocate_streams_sat(c["time"], c["memory"], sat, c["b0"], c["B"], c["P"], c["m_cap"], c["eps"],
                                   c["stall"])
        assert (p.streams, p.minibatch, p.bottleneck) == (c["streams"], c["minibatch"], c["bottleneck"])
    t, m = [0.075, 0.022, 0.013], [12288.0, 12304.0, 24.0]
    ref = q.allocate_streams(t, m, 256.0, 16384, 16, 1e11, 0.0, 2)
    gpu = q.allocate_streams_sat(t, m, [1.08, 2.02, 1.0], 256.0, 16384, 16, 1e11, 0.0, 2)
    assert sum(ref.streams) > sum(gpu.streams) and gpu.streams[2] == 1
    with pytest.raises(q.InvalidInput):
        q.allocate_streams_sat(t, m, [1.0, 1.0], 256.0, 16384, 16, 1e11, 0.0, 2)


def test_allocate_streams_unbounded_cap_documented_divergence():
    """sched.cpp:59 casts floor(M_cap / sum u) to int; for M_cap = 1e18 that is
    undefined (x86: INT_MIN -> InfeasibleConfig, as cmd_bench's own call hits).
    This port clamps to the global batch instead."""
    p = q.allocate_streams([5.0, 7.0, 28.0], [983040.0, 49632.0, 120.0], 16, 128, 16, 1e18, 0.0, 2)
    assert p.minibatch == [128, 128, 128]


def test_compute_calls_fail_loudly_without_gpu():
    torch = pytest.importorskip("torch")
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    with pytest.raises(q.CudaError):
        q.DetectionContext(q.DetectionConfig())


def test_null_context_calls_report_invalid_input():
    """Every context entry point validates its handle before touching CUDA, so
    the reference's InvalidInput convention holds without a device."""
    import ctypes as C
    L = q.lib()
    invalid = 1  # QRM_INVALID_INPUT (include/qrmark_gpu.h)
    assert L.qrm_ctx_set_transfer_split(None, C.c_double(0.5)) == invalid
    assert L.qrm_ctx_set_extractor(None, 0, 7) == invalid
    assert L.qrm_detect_device(None, None, 0, 256, 256, 196608, 0, None, None) == invalid
    assert "null context" in L.qrm_last_error().decode()


def test_multitile_tasks_and_predictors():
    """build_tasks / WarmupStats (sched.cpp:126-155): latency and memory scale with tile area."""
    import numpy as np
    from paper_2509_02447_b200.multitile import (ConstantTilePredictor, ContrastTilePredictor, WarmupStats,
                                                 build_tasks)
    st = WarmupStats(64, 2.0, 12288.0)
    assert st.latency_for(32) == 0.5 and st.latency_for(128) == 8.0 and st.memory_for(80) == 12288.0 * 1.5625
    imgs = [np.zeros((512, 512, 3), np.uint8), np.full((512, 512, 3), 7, np.uint8)]
    assert build_tasks(imgs, ConstantTilePredictor(80), st) == [(0, 80, 3.125, 19200.0), (1, 80, 3.125, 19200.0)]
    flat = ContrastTilePredictor()
    assert flat.select_tile_size(imgs[0]) == 128  # no contrast: the largest tile
    noisy = np.random.default_rng(0).integers(0, 256, (512, 512, 3), dtype=np.uint8)
    assert flat.select_tile_size(noisy) == 32
    with pytest.raises(q.InvalidInput):
        build_tasks(imgs, ConstantTilePredictor(0), st)


@pytest.mark.parametrize("counts,streams,mb,lam,bmin", [({32: 683, 64: 683, 128: 682}, 3, 512, 0.2, 128),
                                                        ({32: 10, 64: 0, 128: 1000}, 2, 256, float("inf"), 64),
                                                        ({64: 4096}, 4, 1024, 0.0, 512)])
def test_multitile_schedule_covers_every_image(counts, streams, mb, lam, bmin):
    """Algorithm 2 over per-size groups (multitile.schedule_groups): the pieces are
    contiguous ranges that cover every image of every group exactly once."""
    from paper_2509_02447_b200.multitile import WarmupStats, schedule_groups
    per_stream, loads = schedule_groups(counts, WarmupStats(64, 0.01, 12288.0), streams, mb, lam, bmin)
    assert len(per_stream) == streams and len(loads) == streams
    for l, c in counts.items():
        covered = sorted((a, a + k) for st in per_stream for (ll, a, k) in st if ll == l)
        pos = 0
        for a, b in covered:
            assert a == pos and b > a
            pos = b
        assert pos == c
