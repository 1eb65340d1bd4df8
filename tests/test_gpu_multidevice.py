"""Multi-device readiness: contexts on every visible GPU, kernel
setup per device, NUMA-local host CPUs. Skips device loops on a one-GPU box."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def test_contexts_on_every_device_decode_identically(qrm, cuda):
    n = cuda.cuda.device_count()
    if n < 2:
        pytest.skip("one visible GPU")
    cfg = qrm.DetectionConfig()
    recs = []
    for d in range(n):
        with cuda.cuda.device(d):
            imgs = qrm.make_corpus(cfg, 1000, 300)
            with qrm.DetectionContext(cfg, device=d) as ctx:
                recs.append(qrm.records_from_device(ctx.detect_device(imgs, first_draw=77)))
    for r in recs[1:]:
        assert np.array_equal(r, recs[0])


def test_device_cpus_and_multi_host_executor(qrm, cuda):
    """qrm_detect_host_multi over every visible device (1 on a one-GPU box) equals
    the single-context result; each device reports its NUMA-local CPUs."""
    n = cuda.cuda.device_count()
    for d in range(n):
        cpus = qrm.device_cpus(d)
        assert all(c >= 0 for c in cpus)
    cfg = qrm.DetectionConfig()
    host = qrm.make_corpus(cfg, 1000, 1000).cpu().numpy()
    ctxs = [qrm.DetectionContext(cfg, device=d) for d in range(n)] + [qrm.DetectionContext(cfg, device=0)]
    try:
        one, _ = ctxs[0].detect_host(host, 5)
        multi, _ = qrm.detect_host_multi(ctxs, host, 5)
        assert np.array_equal(one, multi)
    finally:
        for c in ctxs:
            c.close()
