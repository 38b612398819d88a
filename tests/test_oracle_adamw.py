"""Pins of the AdamW oracle (oracle/adamw.py) against things other than itself.

  * torch.optim.AdamW + torch.nn.utils.clip_grad_norm_ in fp64 over several steps (a library
    routine written independently)                                -> every term, bias correction
  * first step closed form: m_hat = g, v_hat = g^2 -> p - lr * g / (|g| + eps)
                                                                    -> sign, bias correction
  * g = 0: p * (1 - lr wd) exactly, m and v decay geometrically    -> decoupled weight decay
  * clipping: inactive below max_norm; the clipped gradient has norm max_norm (up to the 1e-6)
"""
import numpy as np
import pytest
import torch

from oracle import adamw as OA


@pytest.mark.parametrize("wd,max_norm,gscale", [(0.0, 1.0, 1.0), (0.01, 0.0, 0.5), (0.1, 0.05, 0.25)])
def test_matches_torch_adamw_fp64(wd, max_norm, gscale):
    rng = np.random.default_rng(7)
    n = 1000
    p0 = rng.standard_normal(n)
    lr, b1, b2, eps = 2e-3, 0.9, 0.999, 1e-8
    tp = torch.nn.Parameter(torch.tensor(p0, dtype=torch.float64))
    opt = torch.optim.AdamW([tp], lr=lr, betas=(b1, b2), eps=eps, weight_decay=wd, foreach=False)
    p, m, v = p0.copy(), np.zeros(n), np.zeros(n)
    for t in range(1, 6):
        g = rng.standard_normal(n) * (0.1 * t)
        tp.grad = torch.tensor(g * gscale, dtype=torch.float64)
        if max_norm > 0:
            torch.nn.utils.clip_grad_norm_([tp], max_norm)
        opt.step()
        p, m, v = OA.adamw_step(p, m, v, g, t, lr, b1, b2, eps, wd, gscale, max_norm)
        st = opt.state[tp]
        np.testing.assert_allclose(p, tp.detach().numpy(), rtol=1e-12, atol=1e-14)
        np.testing.assert_allclose(m, st["exp_avg"].numpy(), rtol=1e-12, atol=1e-16)
        np.testing.assert_allclose(v, st["exp_avg_sq"].numpy(), rtol=1e-12, atol=1e-18)


def test_first_step_closed_form():
    g = np.array([3.0, -0.5, 1e-3, 0.0, -2.0])
    p0 = np.array([1.0, 2.0, -1.0, 0.5, 0.0])
    lr, eps = 0.1, 1e-8
    p, m, v = OA.adamw_step(p0, np.zeros(5), np.zeros(5), g, 1, lr, eps=eps)
    np.testing.assert_allclose(p, p0 - lr * g / (np.abs(g) + eps), rtol=1e-15)
    np.testing.assert_allclose(m, 0.1 * g, rtol=1e-15)
    np.testing.assert_allclose(v, 0.001 * g * g, rtol=1e-12)


def test_zero_grad_is_pure_decay():
    p0 = np.array([1.0, -3.0, 0.25])
    m0 = np.array([0.5, 0.0, -0.1])
    v0 = np.array([0.0, 0.0, 0.0])
    lr, wd = 0.01, 0.1
    p, m, v = OA.adamw_step(p0, m0, v0, np.zeros(3), 3, lr, weight_decay=wd)
    # v stays 0: the step is lr * m_hat / eps on entries with m != 0; on m == 0 exactly the decay
    assert p[1] == p0[1] * (1 - lr * wd)
    np.testing.assert_array_equal(m, 0.9 * m0)
    np.testing.assert_array_equal(v, 0.0)


def test_clip_coefficient():
    g = np.array([3.0, 4.0])   # norm 5
    assert OA.clip_coef(g, 10.0) == 1.0
    assert OA.clip_coef(g, 0.0) == 1.0
    c = OA.clip_coef(g, 1.0)
    assert abs(np.linalg.norm(g * c) - 1.0) < 1e-6
