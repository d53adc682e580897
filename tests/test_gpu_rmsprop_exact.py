"""RMSProp bit-exactness at scale (optim.py:107-135 via the oracle's numpy
restatement): the kernels compute each new f32 payload from a MUFU-seeded
approximation of the f64 expression and fall back to the IEEE sqrt /
division only when the approximation cannot prove which float the exact
value rounds to (optim.cu, rms_theta_fast).  These cases aim at that proof:
millions of random rows over wide magnitude ranges, special values, and
second moments solved so that the exact f64 result lands on (or a chosen
distance from) a float rounding midpoint."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

BETA, EPS, LR_SIG, LR_SH = 0.95, 1e-8, 0.1, 0.01


def _random_rows(rng, cap, nsh):
    """theta, v0, g for cap rows of 1 + nsh elements, wide ranges + specials."""
    n = cap * (1 + nsh)
    theta = rng.normal(0, 0.5, n)
    k = rng.integers(0, 8, n)
    theta[k == 0] *= 1e4
    theta[k == 1] *= 1e-30
    theta = theta.astype(np.float32)
    v0 = 10.0 ** rng.uniform(-40, 20, n)
    s = rng.integers(0, 64, n)
    v0[s == 0] = 0.0
    v0[s == 1] = 5e-324
    v0[s == 2] = np.inf
    v0[s == 3] = 1e300
    g = (10.0 ** rng.uniform(-30, 3, n) * rng.choice([-1.0, 1.0], n)).astype(np.float32)
    z = rng.integers(0, 32, n)
    g[z == 0] = 0.0
    g[z == 1] = -0.0
    g[z == 2] = np.float32(1e-45)
    return theta, v0, g


def _midpoint_rows(rng, cap, nsh, lr_sig, lr_sh, eps=EPS):
    """v0 solved so that t = theta - lr g / (sqrt(v) + eps) sits at a float
    rounding midpoint of theta, offset by a relative 2^-k (k in 30..60, both
    signs: inside and just outside the fast path's error bound)."""
    n = cap * (1 + nsh)
    theta = rng.normal(0, 0.5, n).astype(np.float32)
    theta[np.abs(theta) < 1e-3] = np.float32(0.25)
    g = (10.0 ** rng.uniform(-4, 1, n) * rng.choice([-1.0, 1.0], n)).astype(np.float32)
    lr = np.full(n, lr_sh)
    lr[:: 1 + nsh] = lr_sig
    th = theta.astype(np.float64)
    # neighbour on the side the step moves theta to (q = lr g / (...) has g's sign)
    nb = np.nextafter(theta, np.where(g > 0, -np.inf, np.inf).astype(np.float32)).astype(np.float64)
    mid = 0.5 * (th + nb)
    k = rng.integers(30, 61, n).astype(np.float64)
    off = rng.choice([-1.0, 0.0, 1.0], n) * np.ldexp(1.0, -k.astype(np.int64))
    q = (th - mid) * (1.0 + off)
    den = lr * g.astype(np.float64) / q - eps  # sqrt(v_new)
    vn = den * den
    v0 = (vn - (1.0 - BETA) * g.astype(np.float64) ** 2) / BETA
    bad = ~(v0 >= 0) | ~np.isfinite(v0)
    v0[bad] = 1e-6
    return theta, v0, g


def _run(kind, theta, v0, g, cap, nsh, touched, lr_sig=LR_SIG, lr_sh=LR_SH, eps=EPS):
    from paper_2307_15333_b200 import _lib
    dev = torch.device("cuda")
    t2 = theta.reshape(cap, 1 + nsh)
    v2 = v0.reshape(cap, 1 + nsh)
    g2 = g.reshape(cap, 1 + nsh)
    sig = torch.from_numpy(np.ascontiguousarray(t2[:, 0])).to(dev)
    sh = torch.from_numpy(np.ascontiguousarray(t2[:, 1:])).to(dev)
    vs = torch.from_numpy(np.ascontiguousarray(v2[:, 0])).to(dev)
    vh = torch.from_numpy(np.ascontiguousarray(v2[:, 1:])).to(dev)
    gs = torch.from_numpy(np.ascontiguousarray(g2[:, 0])).to(dev)
    gh = torch.from_numpy(np.ascontiguousarray(g2[:, 1:])).to(dev)
    m = torch.from_numpy(touched).to(dev)
    _lib.call(kind, _lib.ptr(sig), _lib.ptr(sh), nsh, nsh, _lib.ptr(vs), _lib.ptr(vh), _lib.ptr(gs), _lib.ptr(gh),
              nsh, _lib.ptr(m), cap, BETA, eps, lr_sig, lr_sh, 0, _lib.stream_ptr())
    torch.cuda.synchronize()
    return sig.cpu().numpy(), sh.cpu().numpy(), vs.cpu().numpy(), vh.cpu().numpy()


def _expect(oracle, theta, v0, g, cap, nsh, touched, lr_sig=LR_SIG, lr_sh=LR_SH, eps=EPS):
    t2 = theta.reshape(cap, 1 + nsh)
    v2 = v0.reshape(cap, 1 + nsh)
    g2 = g.reshape(cap, 1 + nsh).astype(np.float64)
    sig, sh = t2[:, 0].copy(), t2[:, 1:].copy()
    vs, vh = v2[:, 0].copy(), v2[:, 1:].copy()
    with np.errstate(all="ignore"):
        oracle.rmsprop_step(sig, sh, vs, vh, g2[:, 0].copy(), g2[:, 1:].copy(), np.nonzero(touched)[0],
                            beta=BETA, eps=eps, lr_sigma=lr_sig, lr_sh=lr_sh)
    return sig, sh, vs, vh


def _check(got, want):
    for name, a, b in zip(("sigma", "sh", "v_sigma", "v_sh"), got, want):
        # bitwise, NaNs included
        ai = a.view(np.uint32 if a.dtype == np.float32 else np.uint64)
        bi = b.view(np.uint32 if b.dtype == np.float32 else np.uint64)
        bad = np.nonzero(ai.reshape(-1) != bi.reshape(-1))[0]
        assert bad.size == 0, f"{name}: {bad.size} mismatches, first at {bad[:5]}: " \
                              f"{a.reshape(-1)[bad[:5]]} vs {b.reshape(-1)[bad[:5]]}"


@pytest.mark.parametrize("kind", ["dot_rmsprop_step", "dot_rmsprop_step_sparse"])
@pytest.mark.parametrize("nsh", [48, 3])
def test_rmsprop_bit_exact_wide_ranges(oracle, kind, nsh):
    rng = np.random.default_rng(21 + nsh)
    cap = (1 << 17) if nsh == 48 else (1 << 20)
    theta, v0, g = _random_rows(rng, cap, nsh)
    touched = (rng.integers(0, 8, cap) != 0).astype(np.uint8)
    _check(_run(kind, theta, v0, g, cap, nsh, touched), _expect(oracle, theta, v0, g, cap, nsh, touched))


@pytest.mark.parametrize("kind", ["dot_rmsprop_step", "dot_rmsprop_step_sparse"])
@pytest.mark.parametrize("nsh", [48, 3])
def test_rmsprop_bit_exact_at_rounding_midpoints(oracle, kind, nsh):
    rng = np.random.default_rng(31 + nsh)
    cap = (1 << 17) if nsh == 48 else (1 << 20)
    theta, v0, g = _midpoint_rows(rng, cap, nsh, LR_SIG, LR_SH)
    touched = np.ones(cap, np.uint8)
    _check(_run(kind, theta, v0, g, cap, nsh, touched), _expect(oracle, theta, v0, g, cap, nsh, touched))


def test_rmsprop_bit_exact_other_hyperparameters(oracle):
    """lr 1 / eps 0 (sqrt(v) alone in the denominator) and a large eps."""
    rng = np.random.default_rng(41)
    cap, nsh = 1 << 16, 48
    for lr_sig, lr_sh, eps in ((1.0, 1.0, 0.0), (0.5, 2.0, 1e-3), (1e-6, 1e-5, 1e-12)):
        theta, v0, g = _random_rows(rng, cap, nsh)
        touched = np.ones(cap, np.uint8)
        _check(_run("dot_rmsprop_step", theta, v0, g, cap, nsh, touched, lr_sig, lr_sh, eps),
               _expect(oracle, theta, v0, g, cap, nsh, touched, lr_sig, lr_sh, eps))
        theta, v0, g = _midpoint_rows(rng, cap, nsh, lr_sig, lr_sh, eps)
        _check(_run("dot_rmsprop_step", theta, v0, g, cap, nsh, touched, lr_sig, lr_sh, eps),
               _expect(oracle, theta, v0, g, cap, nsh, touched, lr_sig, lr_sh, eps))


@pytest.mark.parametrize("kind", ["dot_rmsprop_step", "dot_rmsprop_step_sparse"])
@pytest.mark.parametrize("nsh", [48, 3])
@pytest.mark.parametrize("eps", [EPS, 0.0])
def test_rmsprop_signed_zeros_and_zero_denominator(oracle, kind, nsh, eps):
    """Every combination of a +-0 payload, a +-0 gradient and v = 0 / > 0 /
    inf: the zero-gradient shortcuts must match the full expression, whose
    -0 - -0 = +0 and (eps = 0, v = 0) 0/0 = NaN the reference keeps."""
    import itertools
    combos = list(itertools.product([0.0, -0.0, 0.5, -0.5], [0.0, -0.0, 1e-3], [0.0, 1e-3, np.inf]))
    per_row = 1 + nsh
    cap = -(-len(combos) * 7 // per_row)
    n = cap * per_row
    theta = np.zeros(n, np.float32)
    g = np.zeros(n, np.float32)
    v0 = np.zeros(n)
    for i in range(n):  # each combination at many positions (sigma column and every quad slot)
        th, gg, vv = combos[i % len(combos)]
        theta[i], g[i], v0[i] = th, gg, vv
    # whole zero-gradient quads too: rows whose gradients are all +0 / all -0
    g2 = g.reshape(cap, per_row)
    g2[::3] = 0.0
    g2[1::3] = -0.0
    touched = np.ones(cap, np.uint8)
    _check(_run(kind, theta, v0, g, cap, nsh, touched, eps=eps),
           _expect(oracle, theta, v0, g, cap, nsh, touched, eps=eps))
