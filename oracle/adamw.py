"""AdamW step over the fine-tune adapters' parameters -- fp64 oracle (TEST INFRASTRUCTURE ONLY).

SURVEY.md §8(f3): "a fused masked AdamW step on the LoRA params (lr 2e-5)" after the per-adapter
gradient reduction.  PAPER.md Table 5 ("Training Args") fixes learning_rate 2e-5 and
gradient_accumulation_steps 4 for the HF Trainer runs but is silent on the optimizer itself; the
reading (R12) is the HF Trainer default, AdamW (decoupled weight decay, Loshchilov &
Hutter) with betas (0.9, 0.999), eps 1e-8, weight_decay 0.0 and global gradient-norm clipping at
max_grad_norm 1.0.  Masking (MixedLoRAModelForTrainer: each trainer updates only its own
adapter) is the caller's choice of which adapters' parameters form the flat buffer.

The update, step t >= 1, every array flat fp64, written in the order of the definition:

    g      = grad * grad_scale                          (grad_scale: 1/world or 1/accumulation)
    norm   = || g ||_2                                  (over the whole buffer)
    g      = g * min(1, max_norm / (norm + 1e-6))       (only if max_norm > 0)
    p      = p * (1 - lr * wd)                          (decoupled weight decay)
    m      = beta1 * m + (1 - beta1) * g
    v      = beta2 * v + (1 - beta2) * g^2
    m_hat  = m / (1 - beta1^t)
    v_hat  = v / (1 - beta2^t)
    p      = p - lr * m_hat / (sqrt(v_hat) + eps)

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may import this module.
"""
from __future__ import annotations

import numpy as np


def clip_coef(g: np.ndarray, max_norm: float) -> float:
    """min(1, max_norm / (||g||_2 + 1e-6)); 1 when clipping is off (max_norm <= 0)."""
    if max_norm <= 0:
        return 1.0
    norm = float(np.sqrt(np.sum(np.asarray(g, np.float64) ** 2)))
    return min(1.0, max_norm / (norm + 1e-6))


def adamw_step(p, m, v, grad, t: int, lr: float, beta1: float = 0.9, beta2: float = 0.999,
               eps: float = 1e-8, weight_decay: float = 0.0, grad_scale: float = 1.0,
               max_norm: float = 0.0):
    """One AdamW step; returns new (p, m, v) as fp64 arrays (inputs are not modified)."""
    p = np.array(p, np.float64)
    m = np.array(m, np.float64)
    v = np.array(v, np.float64)
    g = np.array(grad, np.float64) * grad_scale
    g = g * clip_coef(g, max_norm)
    p = p * (1.0 - lr * weight_decay)
    m = beta1 * m + (1.0 - beta1) * g
    v = beta2 * v + (1.0 - beta2) * g * g
    m_hat = m / (1.0 - beta1 ** t)
    v_hat = v / (1.0 - beta2 ** t)
    p = p - lr * m_hat / (np.sqrt(v_hat) + eps)
    return p, m, v
