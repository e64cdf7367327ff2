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


# ---------------------------------------------------------------------------
# Badly scaled test matrices for the Ozaki engine's accuracy guard.  The four
# structured families restate the reference gallery's definitions
# (/root/reference/pkg/src/cossinm/gallery.py: _frank :68-74, _lehmer
# :110-112, _grcar :127-131, _pascal_lower :143-149), rescaled to a target
# 1-norm the way generate_corpus does (_rescaled, gallery.py:182-183).

def gallery_pascal_lower(n):
    m = np.zeros((n, n))
    m[:, 0] = 1.0
    for i in range(1, n):
        m[i, 1:i + 1] = m[i - 1, 0:i] + m[i - 1, 1:i + 1]
    return m


def gallery_frank(n):
    i, j = np.indices((n, n))
    return np.where(j >= i - 1, n - np.maximum(i, j), 0).astype(np.float64)


def gallery_lehmer(n):
    i, j = np.indices((n, n)) + 1
    return np.minimum(i, j) / np.maximum(i, j)


def gallery_grcar(n):
    m = -np.eye(n, k=-1)
    for k in range(4):
        m += np.eye(n, k=k)
    return m


def graded(rng, n, spread):
    """D B D^-1 with D = diag(logspace(0, log10 spread)) and B ~ N(0,1):
    rows and columns graded over `spread` (entries span spread^2)."""
    d = np.logspace(0.0, np.log10(spread), n)
    return (d[:, None] * rng.standard_normal((n, n))) / d[None, :]


def rescaled(m, target):
    """gallery._rescaled: m * (target / norm1(m))."""
    return m * (target / np.abs(m).sum(axis=0).max())


def permuted_noise(fn, a, rng):
    """The reference's own noise floor for input `a`: run the
    oracle `fn` (returning (cos, sin, ...)) on P a P^T and undo P -- the
    same matrix function with every GEMM summed in a different order.
    Returns (outputs of fn(a), max relative 1-norm distance of the pair)."""
    out = fn(a)
    perm = rng.permutation(a.shape[-1])
    inv = np.argsort(perm)
    outp = fn(a[np.ix_(perm, perm)])
    noise = 0.0
    for x, xp in zip(out[:2], outp[:2]):
        noise = max(noise, rel1(xp[np.ix_(inv, inv)], x))
    return out, noise
