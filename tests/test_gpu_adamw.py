"""GPU parity of the AdamW step (kernels_opt.cu) against the fp64 oracle
(oracle/adamw.py), through the C ABI (smlm_adamw_step).

Tolerance (R12): the kernel computes in fp32, so parameters and moments must agree with
the fp64 oracle to rtol 2e-5 (a few fp32 ulps through ~10 dependent operations, plus the fp32
sum of squares of the clip pass); the bf16 working copy must equal bf16(fp32 parameter) exactly
and the oracle to within one bf16 ulp.  The clip coefficient and everything else is bitwise
reproducible run to run."""
import numpy as np
import pytest
import torch

import synth
from oracle import adamw as OA

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def S():
    from paper_2511_00101_b200 import smlm
    return smlm


def _run(S, p, m, v, g, t, with_bf16=True, ws=True, **hp):
    dev = torch.device("cuda", 0)
    P, M, V, G = (x.clone().to(dev) for x in (p, m, v, g))
    PB = torch.empty(p.numel(), dtype=torch.bfloat16, device=dev) if with_bf16 else None
    W = torch.empty(max(S.smlm_adamw_workspace_size() // 4, 1), dtype=torch.float32, device=dev) if ws else None
    S.smlm_adamw_step(P, M, V, G, PB, t, ws=W, **hp)
    torch.cuda.synchronize()
    return P.cpu(), M.cpu(), V.cpu(), G.cpu(), None if PB is None else PB.cpu()


def _check(out, ref, inp, gscale=1.0, lr=0.0, wd=0.0, beta1=0.9, tol=2e-5):
    """Elementwise |got - oracle| <= tol * (magnitude of the terms that form the result): the
    parameter update can cancel the decayed parameter, so the bound uses |p decay| + |update|."""
    P, M, V = (x.double().numpy() for x in out[:3])
    p, m, v = ref
    p0, m0, _, g = (np.asarray(x, np.float64) for x in inp)
    decayed = p0 * (1.0 - lr * wd)
    sp = np.abs(decayed) + np.abs(p - decayed)
    sm = beta1 * np.abs(m0) + (1.0 - beta1) * np.abs(g) * gscale
    for got, exp, sc in ((P, p, sp), (M, m, sm), (V, v, np.abs(v))):
        bad = np.abs(got - exp) > tol * sc + 1e-30
        assert not bad.any(), (np.flatnonzero(bad)[:5], got[bad][:5], exp[bad][:5])


@pytest.mark.parametrize("n", [1, 3, 4, 1001, 65536 + 5, 3 * 2**20 + 3])
@pytest.mark.parametrize("t", [1, 7])
def test_adamw_parity(S, n, t):
    p, m, v, g = synth.draw_adamw_state(n + 17 * t, n, step=t)
    hp = dict(lr=2e-5, beta1=0.9, beta2=0.999, eps=1e-8, weight_decay=0.01, grad_scale=0.25, max_grad_norm=0.0)
    out = _run(S, p, m, v, g, t, **hp)
    ref = OA.adamw_step(p.numpy(), m.numpy(), v.numpy(), g.numpy(), t, 2e-5, 0.9, 0.999, 1e-8, 0.01, 0.25, 0.0)
    _check(out, ref, (p, m, v, g), gscale=0.25, lr=2e-5, wd=0.01)
    # bf16 copy: exactly the conversion of the kernel's own fp32, within 1 ulp of the oracle's
    assert torch.equal(out[4], out[0].to(torch.bfloat16))
    ref_b = torch.from_numpy(ref[0]).to(torch.float32).to(torch.bfloat16).float()
    ulp = torch.from_numpy(np.abs(ref[0])).float().clamp_min(1e-30) * 2.0 ** -7
    assert bool(((out[4].float() - ref_b).abs() <= ulp).all())
    assert torch.equal(out[3], g)   # zero_grad off: gradient untouched


@pytest.mark.parametrize("max_norm", [1.0, 1e-3, 1e6])
def test_adamw_clip(S, max_norm):
    n = 2**20 + 9
    p, m, v, g = synth.draw_adamw_state(3, n, step=3)
    g = g * 10.0   # ||g|| ~ 10 so max_norm 1 and 1e-3 clip, 1e6 does not
    hp = dict(lr=1e-3, beta1=0.9, beta2=0.999, eps=1e-8, weight_decay=0.0, grad_scale=0.5, max_grad_norm=max_norm,
              zero_grad=True)
    out = _run(S, p, m, v, g, 3, **hp)
    ref = OA.adamw_step(p.numpy(), m.numpy(), v.numpy(), g.numpy(), 3, 1e-3, 0.9, 0.999, 1e-8, 0.0, 0.5, max_norm)
    _check(out, ref, (p, m, v, g), gscale=0.5, lr=1e-3)
    assert bool((out[3] == 0).all())   # zero_grad
    # bitwise reproducible (fixed reduction order)
    out2 = _run(S, p, m, v, g, 3, **hp)
    for a, b in zip(out[:3], out2[:3]):
        assert torch.equal(a, b)


def test_adamw_multistep_matches_oracle(S):
    """Five steps with the moments carried on the device (state never leaves the GPU)."""
    n = 40000 + 3
    p, m, v, _ = synth.draw_adamw_state(11, n, step=1)
    dev = torch.device("cuda", 0)
    P, M, V = p.to(dev), m.to(dev), v.to(dev)
    G = torch.empty(n, device=dev)
    W = torch.empty(S.smlm_adamw_workspace_size() // 4, device=dev)
    rp, rm, rv = p.numpy(), m.numpy(), v.numpy()
    for t in range(1, 6):
        g = synth.draw_adamw_state(100 + t, n)[3]
        G.copy_(g)
        S.smlm_adamw_step(P, M, V, G, None, t, 2e-5, weight_decay=0.1, max_grad_norm=1.0, ws=W)
        inp = (rp, rm, rv, g.numpy())
        rp, rm, rv = OA.adamw_step(rp, rm, rv, g.numpy(), t, 2e-5, weight_decay=0.1, max_norm=1.0)
        torch.cuda.synchronize()
        # compare every step (the device state carries the kernel's own rounding forward)
        _check((P.cpu(), M.cpu(), V.cpu()), (rp, rm, rv), inp, lr=2e-5, wd=0.1, tol=5e-5)
        rp, rm, rv = (x.cpu().double().numpy() for x in (P, M, V))


def test_adamw_errors(S):
    dev = torch.device("cuda", 0)
    x = torch.zeros(64, device=dev)
    with pytest.raises(S.SmlmError) as e:
        S.smlm_adamw_step(x, x.clone(), x.clone(), x.clone(), None, 0, 1e-3)           # step 0
    assert e.value.code == S.SMLM_E_INVALID
    with pytest.raises(S.SmlmError) as e:
        S.smlm_adamw_step(x, x.clone(), x.clone(), x.clone(), None, 1, 1e-3, beta1=1.0)
    assert e.value.code == S.SMLM_E_INVALID
    with pytest.raises(S.SmlmError) as e:
        S.smlm_adamw_step(x[1:], x.clone()[1:], x.clone()[1:], x.clone()[1:], None, 1, 1e-3)   # misaligned
    assert e.value.code == S.SMLM_E_INVALID
    with pytest.raises(S.SmlmError) as e:
        S.smlm_adamw_step(x, x.clone(), x.clone(), x.clone(), None, 1, 1e-3, max_grad_norm=1.0)   # no workspace
    assert e.value.code == S.SMLM_E_WORKSPACE
    # n = 0 is a no-op
    e0 = torch.zeros(0, device=dev)
    S.smlm_adamw_step(e0, e0, e0, e0, None, 1, 1e-3)


def test_adapter_params_train_step(S):
    """optim.AdapterParams + AdamW: the SMLM backward writes dA/dB into the flat gradient, one
    AdamW launch updates the master weights, and the pool sees the new bf16 values."""
    from paper_2511_00101_b200.optim import AdapterParams, AdamW
    in_f, out_f, r = 256, 192, 16
    gen = torch.Generator().manual_seed(5)
    w = synth.draw_weights(gen, in_f, out_f, r, 2)
    dev = torch.device("cuda", 0)
    store = AdapterParams([(r, in_f, out_f)] * 2, device=dev)
    for k in range(2):
        store.load(k, w.A[k].float(), w.B[k].float())
    pool = S.Pool(in_f, out_f, r, 4, S.SMLM_BF16, 0)
    slots = [pool.register(store.A(k), store.B(k), 2.0) for k in range(2)]
    for k, sl in enumerate(slots):
        pool.set_grad(sl, store.dA(k), store.dB(k))
    batch = synth.batch_from_lengths([40, 24], slots, [synth.FINETUNE] * 2)
    b = S.Batch.from_synth(batch)
    X = torch.randn(64, in_f, generator=gen).to(torch.bfloat16).to(dev)
    W = (torch.randn(out_f, in_f, generator=gen) / 16).to(torch.bfloat16).to(dev)
    dY = torch.randn(64, out_f, generator=gen).to(torch.bfloat16).to(dev)
    V = torch.empty(64, r, dtype=torch.bfloat16, device=dev)
    Y = pool.forward(b, X, W, V_save=V)
    pool.backward(b, X, W, dY, V, None)
    g_host = store.grad.cpu().clone()
    p_host = store.master.cpu().clone()
    opt = AdamW(store, lr=1e-3, max_grad_norm=1.0)
    opt.step()
    torch.cuda.synchronize()
    # one job per adapter (the default): each clips by its own norm (optim.py)
    for j, (lo, hi) in store.job_range.items():
        n = hi - lo
        ref_p, _, _ = OA.adamw_step(p_host[lo:hi].numpy(), np.zeros(n), np.zeros(n), g_host[lo:hi].numpy(), 1, 1e-3,
                                    max_norm=1.0)
        _check((store.master[lo:hi].cpu(), torch.zeros(n), torch.zeros(n)), (ref_p, np.zeros(n), np.zeros(n)),
               (p_host[lo:hi].numpy(), np.zeros(n), None, g_host[lo:hi].numpy()), lr=1e-3)
    assert bool((store.grad == 0).all())
    assert torch.equal(store.bf16, store.master.to(torch.bfloat16))
    # the next forward uses the updated adapter (borrowed bf16 views)
    Y2 = pool.forward(b, X, W)
    assert not torch.equal(Y, Y2)
    pool.close()


def test_adamw_per_job_clip_and_steps(S):
    """Per-job optimizer state (Loquetier runs one HF Trainer per fine-tune job): a job
    with a huge gradient does not shrink another job's update, and a job that steps less often
    keeps its own step count (bias correction) -- against the fp64 oracle per job."""
    from paper_2511_00101_b200.optim import AdapterParams, AdamW
    dev = torch.device("cuda", 0)
    store = AdapterParams([(8, 64, 48), (8, 64, 48), (16, 128, 64)], device=dev, jobs=[0, 0, 1])
    assert store.job_range[0][1] == store.job_range[1][0]
    g = torch.Generator(device=dev).manual_seed(9)
    store.master.copy_(torch.randn(store.n, device=dev, generator=g) * 0.02)
    opt = AdamW(store, lr=1e-3, max_grad_norm=1.0)
    host = {j: (store.master[lo:hi].double().cpu().numpy(), np.zeros(hi - lo), np.zeros(hi - lo))
            for j, (lo, hi) in store.job_range.items()}
    steps = {0: 0, 1: 0}
    for it in range(3):
        jobs = [0, 1] if it != 1 else [1]          # job 0 accumulates over two micro-batches once
        for j in jobs:
            lo, hi = store.job_range[j]
            scale = 100.0 if j == 1 else 1e-3          # job 1: a huge gradient (clipped hard)
            store.grad[lo:hi].copy_(torch.randn(hi - lo, device=dev, generator=g) * scale)
        gh = store.grad.double().cpu().numpy().copy()
        opt.step(jobs)
        torch.cuda.synchronize()
        for j in jobs:
            lo, hi = store.job_range[j]
            steps[j] += 1
            p0, m0, v0 = host[j]
            ref = OA.adamw_step(p0, m0, v0, gh[lo:hi], steps[j], 1e-3, max_norm=1.0)
            _check((store.master[lo:hi].cpu(), store.exp_avg[lo:hi].cpu(), store.exp_avg_sq[lo:hi].cpu()), ref,
                   (p0, m0, v0, gh[lo:hi]), lr=1e-3)
            host[j] = tuple(np.asarray(x, np.float64) for x in (store.master[lo:hi].double().cpu().numpy(),
                                                                store.exp_avg[lo:hi].double().cpu().numpy(),
                                                                store.exp_avg_sq[lo:hi].double().cpu().numpy()))
    assert opt.t == {0: 2, 1: 3}


def test_adamw_full_size_sampled(S):
    """The bench's F3 workload size (4 fine-tune adapters x r=16 x 7 Llama-3-8B projections x 32
    layers = 167.8 M parameters) in the launch configuration bench.py times (clip 1.0, zero_grad,
    bf16 copy): sampled elements against the oracle, with the clip coefficient of the oracle
    computed in fp64 over the whole gradient."""
    n = 4 * synth.lora_param_count(16) * 32
    dev = torch.device("cuda", 0)
    g = torch.Generator(device=dev).manual_seed(123)
    P = torch.randn(n, device=dev, generator=g) * 0.02
    M = torch.randn(n, device=dev, generator=g) * 1e-4
    V = (torch.randn(n, device=dev, generator=g) * 1e-6).abs()
    G = torch.randn(n, device=dev, generator=g) * 1e-3
    idx = torch.randint(0, n, (200000,), device=dev, generator=g)
    p0, m0, v0, g0 = (x[idx].double().cpu().numpy() for x in (P, M, V, G))
    gnorm = float(torch.linalg.vector_norm(G.double()).item())
    PB = torch.empty(n, dtype=torch.bfloat16, device=dev)
    W = torch.empty(S.smlm_adamw_workspace_size() // 4, device=dev)
    S.smlm_adamw_step(P, M, V, G, PB, 5, 2e-5, weight_decay=0.01, max_grad_norm=1.0, zero_grad=True, ws=W)
    torch.cuda.synchronize()
    coef = min(1.0, 1.0 / (gnorm + 1e-6))
    ref = OA.adamw_step(p0, m0, v0, g0 * coef, 5, 2e-5, weight_decay=0.01)   # clip applied with the full norm
    got = (P[idx].cpu(), M[idx].cpu(), V[idx].cpu())
    _check(got, ref, (p0, m0, v0, g0 * coef), lr=2e-5, wd=0.01)
    assert bool((G[idx] == 0).all())
    assert torch.equal(PB[idx], P[idx].to(torch.bfloat16))
