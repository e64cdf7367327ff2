"""Helpers shared by the test modules (comparisons, seeded generators)."""
import numpy as np


def rel1(x, ref):
    """Relative 1-norm difference ||x - ref||_1 / ||ref||_1 (0-safe)."""
    x = np.asarray(x, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    if x.size == 0:
        return 0.0
    d = np.abs(x - ref).sum(axis=-2).max()
    r = np.abs(ref).sum(axis=-2).max()
    return float(d / r) if r > 0 else float(d)


def pair_close(x, ref, partner_ref, tol):
    """Parity test for one output of a (cos, sin) pair: relative 1-norm
    difference <= tol, or -- when the reference output is itself pure
    cancellation residue (sin(pi I) ~ 1e-16) -- difference <= tol on the
    pair's scale ||partner||_1.  Returns (ok, measured)."""
    r = rel1(x, ref)
    if r <= tol:
        return True, r
    x = np.asarray(x, dtype=np.float64)
    d = float(np.abs(x - ref).sum(axis=-2).max()) if x.size else 0.0
    scale = float(np.abs(np.asarray(partner_ref, dtype=np.float64)).sum(axis=-2).max())
    return d <= tol * scale, r


def pythagorean_residual(c, s):
    """||C^2 + S^2 - I||_1 (reported beside the parity numbers)."""
    c = np.asarray(c, dtype=np.float64)
    s = np.asarray(s, dtype=np.float64)
    r = c @ c + s @ s - np.eye(c.shape[-1])
    return float(np.abs(r).sum(axis=0).max())


def cfg2_like(rng, count, n=64, lo=-3.0, hi=2.0):
    """BASELINE configs[1]: N(0,1) entries, 1-norm log-uniform in
    [10^lo, 10^hi]."""
    g = rng.standard_normal((count, n, n))
    tgt = 10.0 ** rng.uniform(lo, hi, count)
    nrm = np.abs(g).sum(axis=1).max(axis=1)
    return g * (tgt / nrm)[:, None, None]


def cfg3_like(rng, count, n=256, lo=-2.0, hi=np.log10(50.0)):
    """BASELINE configs[2]: U(-1,1) entries, 1-norm log-uniform in
    [1e-2, 50], stored as float32."""
    g = rng.uniform(-1.0, 1.0, (count, n, n))
    tgt = 10.0 ** rng.uniform(lo, hi, count)
    nrm = np.abs(g).sum(axis=1).max(axis=1)
    return (g * (tgt / nrm)[:, None, None]).astype(np.float32)


def laplacian_wave(rng, count, n):
    """BASELINE configs[3]: tridiag(-1,2,-1)(n+1)^2 + diag(U(0,10)); t
    log-uniform in [1e-4, 1e-1]."""
    lap = (np.diag(2.0 * np.ones(n)) - np.diag(np.ones(n - 1), 1)
           - np.diag(np.ones(n - 1), -1)) * float((n + 1) ** 2)
    v = rng.uniform(0.0, 10.0, (count, n))
    a = lap[None, :, :] + v[:, :, None] * np.eye(n)[None, :, :]
    t = 10.0 ** rng.uniform(-4.0, -1.0, count)
    return a, t
