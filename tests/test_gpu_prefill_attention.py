"""Corrected prefill attention on the tensor cores (kvlc_corrected_attention) against the
float64 reference forms (corrected_attention_quadratic, attention.py:99-116), whose shim
kernel is pinned to the golden vectors (tests/test_gpu_ref.py)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

import paper_2510_05373_b200 as qk  # noqa: E402
from paper_2510_05373_b200.attention import corrected_attention_batched  # noqa: E402

D = 128


def _case(heads, n, seed, qscale=1.0):
    g = qk.rng(seed)
    q = g.standard_normal((heads, n, D)) * qscale
    kq = g.standard_normal((heads, n, D))
    ke = 0.3 * g.standard_normal((heads, n, D))
    vq = g.standard_normal((heads, n, D))
    return q, kq, ke, vq


@pytest.mark.parametrize("adapter", [False, True])
@pytest.mark.parametrize("n", [1, 70, 300])
def test_matches_reference_forms(adapter, n):
    heads = 3
    q, kq, ke, vq = _case(heads, n, 100 + n)
    ads = [qk.CorrectionAdapter.initialize(D, 256, seed=h) for h in range(heads)] if adapter else None
    out = corrected_attention_batched(q, kq, ke, vq, ads).cpu().numpy()
    for h in range(heads):
        ref = qk.corrected_attention_quadratic(q[h], kq[h], ke[h], vq[h], ads[h] if ads else None)
        err = np.abs(out[h] - ref).max() / np.abs(ref).max()
        assert err <= 1e-4, (h, err)


def test_correction_dominated_and_large_logits():
    """Logits of +-300 (the reference's raw exponentials in float64): the max(0, M) frame keeps
    both the softmax-dominated rows and the correction-dominated rows exact."""
    heads, n = 2, 200
    for sign in (1.0, -1.0):
        q, kq, ke, vq = _case(heads, n, 7, qscale=1.0)
        kq = np.abs(kq) * sign
        q = np.abs(q) * 30.0   # q . k / sqrt(128) ~ +-300
        ads = [qk.CorrectionAdapter.initialize(D, 256, seed=h) for h in range(heads)]
        out = corrected_attention_batched(q, kq, ke, vq, ads).cpu().numpy()
        for h in range(heads):
            ref = qk.corrected_attention_quadratic(q[h], kq[h], ke[h], vq[h], ads[h])
            assert np.isfinite(out[h]).all()
            assert np.abs(out[h] - ref).max() <= 1e-4 * np.abs(ref).max(), (sign, h)


def test_recurrent_form_same_outputs():
    q, kq, ke, vq = _case(1, 129, 3)
    ad = qk.CorrectionAdapter.initialize(D, 256, seed=0)
    out = corrected_attention_batched(q, kq, ke, vq, [ad]).cpu().numpy()[0]
    ref = qk.corrected_attention_recurrent(q[0], kq[0], ke[0], vq[0], ad)
    assert np.abs(out - ref).max() <= 1e-4 * np.abs(ref).max()
