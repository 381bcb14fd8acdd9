"""K5 statistics -> the reference indicator.  OpStats fields collected on the
device (qsync_tensor_stats) and by the oracle for the same activation / weight /
gradient tensors are fed to the REFERENCE's sigma_fwd / sigma_bwd / omega
(indicator.cpp:65-132) and reduce_stats (profile.cpp:134-162); the device-fed
scores must match the CPU-fed ones (north star: 1e-3; observed ~1e-12)."""
import numpy as np
import pytest
import torch

from paper_2407_02327_b200 import ops

pytestmark = pytest.mark.gpu


def _opstats(act, w, grad, stats_fn):
    sa, sw, sg = stats_fn(act), stats_fn(w), stats_fn(grad)
    # profile.hpp:95-108 field order: norm_w_sq, norm_act_sq, norm_grad_act_sq,
    # norm_grad_act_hat_sq, d_act, d_w, d_grad, q_act, q_w, e_act, e_w, e_grad
    return np.array([sw[0], sa[0], sg[0], 0.0, sa[4], sw[4], sg[4], sa[2], sw[2], sa[3], sw[3],
                     sg[3]], np.float64)


@pytest.mark.parametrize("shape", [((4096, 768), (2304, 768)), ((64, 1024), (1024, 1024)),
                                   ((333, 3072), (768, 3072))])
def test_device_stats_drive_reference_indicator(shape, cpuref, reflib):
    (M, K), (N, _) = shape
    rng = np.random.default_rng(M + N)
    act = rng.normal(size=(M, K)).astype(np.float32)
    w = (rng.uniform(-1, 1, size=(N, K)) / np.sqrt(K)).astype(np.float32)
    grad = (rng.normal(size=(M, N)) * 1e-3).astype(np.float32)

    def dev(x):
        t = torch.from_numpy(x).cuda()
        return ops.tensor_stats(t).cpu().numpy()

    v_dev = _opstats(act, w, grad, dev)
    v_cpu = _opstats(act, w, grad, cpuref.tensor_stats)
    mask = 0xFFF & ~(1 << 3)  # no separately profiled grad-hat norm (falls back, indicator.cpp:57-61)
    for p in (0, 1, 2):
        for pf in (0, 1):
            for which in (0, 1):
                a = reflib.sigma(which, v_dev, mask, p, pf)
                b = reflib.sigma(which, v_cpu, mask, p, pf)
                assert a == pytest.approx(b, rel=1e-9, abs=0.0)
        wa = reflib.omega(v_dev, mask, 1, 3, 12, 0, 32, p)
        wb = reflib.omega(v_cpu, mask, 1, 3, 12, 0, 32, p)
        assert wa == pytest.approx(wb, rel=1e-9, abs=0.0)
    # exact fields
    for i in (4, 5, 6, 7, 8, 9, 10, 11):
        assert v_dev[i] == v_cpu[i]


def test_device_stats_window_reduce_reference(cpuref, reflib):
    """Per-iteration device snapshots -> reference reduce_stats (mean of the FIRST W)."""
    rng = np.random.default_rng(3)
    snaps_dev, snaps_cpu = [], []
    for it in range(6):
        act = (rng.normal(size=(256, 768)) * (1 + it)).astype(np.float32)
        w = rng.uniform(-0.1, 0.1, size=(768, 768)).astype(np.float32)
        g = (rng.normal(size=(256, 768)) * 1e-2).astype(np.float32)
        snaps_dev.append(_opstats(act, w, g, lambda x: ops.tensor_stats(torch.from_numpy(x).cuda()).cpu().numpy()))
        snaps_cpu.append(_opstats(act, w, g, cpuref.tensor_stats))
    masks = np.full(6, 0xFFF & ~(1 << 3), np.uint32)
    for window in (1, 4, 50):
        a, ma = reflib.reduce_stats(np.array(snaps_dev), masks, window)
        b, mb = reflib.reduce_stats(np.array(snaps_cpu), masks, window)
        assert ma == mb
        np.testing.assert_allclose(a, b, rtol=1e-10, atol=0.0)
