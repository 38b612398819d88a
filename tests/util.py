"""Shared test helpers: the parity metric (SURVEY.md §8(c) "Parity criteria")."""
import numpy as np

BF16_TOL = 2e-2   # BASELINE.json north_star: max relative error 2e-2 for bf16 inputs, fp32 accumulate
FP32_TOL = 1e-5   # BASELINE.json north_star: 1e-5 in the fp32 test mode


def to64(t):
    import torch
    if isinstance(t, torch.Tensor):
        return t.detach().to("cpu", torch.float64).numpy()
    return np.asarray(t, np.float64)


def parity_err(got, ref) -> float:
    """max_i |g_i - r_i| / max(|r_i|, rms(r)) with rms over the whole compared tensor.

    Reading of "max relative error" (reading R4): a pure elementwise relative error
    is unusable near zero-valued reference entries, so the denominator is floored at the rms.
    """
    g = to64(got).ravel()
    r = to64(ref).ravel()
    if r.size == 0:
        return 0.0
    rms = float(np.sqrt(np.mean(r * r)))
    den = np.maximum(np.abs(r), rms if rms > 0 else 1.0)
    return float(np.max(np.abs(g - r) / den))


def normwise_err(got, ref) -> float:
    g = to64(got).ravel()
    r = to64(ref).ravel()
    n = np.linalg.norm(r)
    return float(np.linalg.norm(g - r) / (n if n > 0 else 1.0))
