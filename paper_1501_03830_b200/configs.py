"""Seeded synthetic inputs for the BASELINE.json configurations.

The paper's matrices (naphthalene / GaAs / BN) are unpublished, so the
BASELINE configs define synthetic recipes; these generators implement them:

  cfg0  real n=512:     Haar U1, U2; s, d ~ U[1,10]; S = U1 diag(s) U1^T,
                        D = U2 diag(d) U2^T; A = (S+D)/2, B = (S-D)/2
                        (so M = A+B = S and K = A-B = D); dipoles d ~ N(0,1)^n
  cfg1  complex n=2048: A = U diag(a) U^H, U Haar-unitary, a ~ U[2,10];
                        B = (G+G^T)/2, G complex normal, ||B||_2 = 1
  cfg2  cfg0 recipe at n=16384 with s, d log-uniform on [0.1, 100]
  cfg3  cfg1 recipe at n=16384 with ||B||_2 = 0.9 min(a)
  cfg4  real n=65536; s, d = 256 clusters x 256 values, centres U[1,10],
        intra-cluster relative spread 1e-6

Dipoles follow the reference API (length 2n, spectra.py:135-136): the
n-vector d drawn by the config is passed as [d; conj(d)] (D5).

numpy generators (PCG64, seed = config index by default) produce the small
parity cases; ``torch_real_operator`` builds the large bench inputs on the GPU
with the same recipe (torch's Philox stream, so the draws differ from numpy's
at equal seed -- stated in the bench line).
"""
from __future__ import annotations

import numpy as np

CONFIGS = {
    0: dict(kind="real", n=512, spectrum="uniform", lo=1.0, hi=10.0, sigma=0.05, grid=2000),
    1: dict(kind="complex", n=2048, lo=2.0, hi=10.0, bnorm="one", sigma=0.05, grid=2000),
    2: dict(kind="real", n=16384, spectrum="loguniform", lo=0.1, hi=100.0, sigma=0.05,
            grid=2000, tile=512),
    3: dict(kind="complex", n=16384, lo=2.0, hi=10.0, bnorm="0.9min", sigma=0.05, grid=2000),
    4: dict(kind="real", n=65536, spectrum="clustered", lo=1.0, hi=10.0, sigma=0.05,
            grid=2000, tile=1024),
}


def haar_orthogonal(rng, n):
    q, r = np.linalg.qr(rng.standard_normal((n, n)))
    return q * np.sign(np.diagonal(r))


def haar_unitary(rng, n):
    g = rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))
    q, r = np.linalg.qr(g)
    d = np.diagonal(r)
    return q * (d / np.abs(d))


def draw_spectrum(rng, n, spectrum, lo, hi, clusters=256, spread=1e-6):
    if spectrum == "uniform":
        return rng.uniform(lo, hi, n)
    if spectrum == "loguniform":
        return np.exp(rng.uniform(np.log(lo), np.log(hi), n))
    if spectrum == "clustered":
        per = max(1, n // clusters)
        nc = int(np.ceil(n / per))
        centres = rng.uniform(lo, hi, nc)
        vals = np.repeat(centres, per)[:n]
        return vals * (1.0 + spread * rng.uniform(-1.0, 1.0, n))
    raise ValueError(spectrum)


def real_operator(n, seed=0, spectrum="uniform", lo=1.0, hi=10.0):
    """(A, B, dipole n-vector) for the real recipes (cfg0 / cfg2 / cfg4)."""
    rng = np.random.default_rng(seed)
    u1 = haar_orthogonal(rng, n)
    u2 = haar_orthogonal(rng, n)
    s = draw_spectrum(rng, n, spectrum, lo, hi)
    d = draw_spectrum(rng, n, spectrum, lo, hi)
    S = (u1 * s) @ u1.T
    D = (u2 * d) @ u2.T
    S = 0.5 * (S + S.T)
    D = 0.5 * (D + D.T)
    dip = rng.standard_normal(n)
    return 0.5 * (S + D), 0.5 * (S - D), dip


def spectral_norm(b, iters=200, seed=0):
    """Power iteration on B^H B (BASELINE cfg3 recipe)."""
    x = np.random.default_rng(seed).standard_normal(b.shape[0]).astype(np.complex128)
    x /= np.linalg.norm(x)
    val = 0.0
    for _ in range(iters):
        y = b.conj().T @ (b @ x)
        val = np.linalg.norm(y)
        if val == 0.0:
            return 0.0
        x = y / val
    return float(np.sqrt(val))


def complex_operator(n, seed=1, lo=2.0, hi=10.0, bnorm="one"):
    """(A, B, dipole n-vector) for the complex recipes (cfg1 / cfg3)."""
    rng = np.random.default_rng(seed)
    u = haar_unitary(rng, n)
    a_vals = rng.uniform(lo, hi, n)
    A = (u * a_vals) @ u.conj().T
    A = 0.5 * (A + A.conj().T)
    g = rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))
    B = 0.5 * (g + g.T)
    target = 1.0 if bnorm == "one" else 0.9 * float(np.min(a_vals))
    B = B * (target / np.linalg.norm(B, 2) if n <= 4096 else target / spectral_norm(B))
    dip = rng.standard_normal(n) + 1j * rng.standard_normal(n)
    return A, B, dip, np.sort(a_vals)[::-1]


def dipole_2n(d):
    """Reference-API dipole of length 2n from the config's n-vector (D5)."""
    d = np.asarray(d, dtype=np.complex128)
    return np.concatenate([d, d.conj()])


def config_operator(idx, n=None, seed=None):
    """Generate config ``idx`` (optionally at a reduced n for parity tests)."""
    c = CONFIGS[idx]
    n = c["n"] if n is None else n
    seed = idx if seed is None else seed
    if c["kind"] == "real":
        a, b, d = real_operator(n, seed, c["spectrum"], c["lo"], c["hi"])
        return a, b, dipole_2n(d)
    a, b, d, _ = complex_operator(n, seed, c["lo"], c["hi"], c["bnorm"])
    return a, b, dipole_2n(d)


def torch_real_operator(n, seed=2, spectrum="loguniform", lo=0.1, hi=100.0, device="cuda"):
    """GPU generator for the large real configs: returns M = A+B = S and
    K = A-B = D directly (column-major == row-major for symmetric matrices)
    plus the dipole n-vector.  Generation (QR via torch) is off the timed
    solve path."""
    import torch
    g = torch.Generator(device=device)
    g.manual_seed(seed)

    def haar():
        z = torch.randn(n, n, dtype=torch.float64, device=device, generator=g)
        q, r = torch.linalg.qr(z)
        return q * torch.sign(torch.diagonal(r))

    def spec():
        u = torch.rand(n, dtype=torch.float64, device=device, generator=g)
        if spectrum == "uniform":
            return lo + (hi - lo) * u
        if spectrum == "loguniform":
            return torch.exp(np.log(lo) + (np.log(hi) - np.log(lo)) * u)
        if spectrum == "clustered":  # cfg4 recipe: 256 clusters, 1e-6 relative spread
            per = max(1, n // 256)
            nc = -(-n // per)
            centres = lo + (hi - lo) * torch.rand(nc, dtype=torch.float64, device=device, generator=g)
            vals = centres.repeat_interleave(per)[:n]
            return vals * (1.0 + 1e-6 * (2.0 * u - 1.0))
        raise ValueError(spectrum)

    u1 = haar()
    s = spec()
    S = (u1 * s) @ u1.T
    del u1
    u2 = haar()
    d = spec()
    D = (u2 * d) @ u2.T
    del u2
    S = 0.5 * (S + S.T)
    D = 0.5 * (D + D.T)
    dip = torch.randn(n, dtype=torch.float64, device=device, generator=g)
    return S, D, dip


def torch_complex_operator(n, seed=3, lo=2.0, hi=10.0, bnorm="0.9min", device="cuda"):
    """GPU generator for the complex recipes (cfg1 / cfg3): A = U diag(a) U^H
    (U Haar-unitary via QR of a complex Ginibre matrix with phase fix),
    B = (G + G^T) / 2 rescaled to ||B||_2 = 1 or 0.9 min(a) (spectral norm by
    power iteration on B^H B, as the host generator).  Returns torch
    complex128 A, B (row-major), the dipole n-vector and a descending.  Off
    the timed path; torch's Philox stream, so draws differ from numpy's."""
    import torch
    g = torch.Generator(device=device)
    g.manual_seed(seed)

    def cnormal(*shape):
        re = torch.randn(*shape, dtype=torch.float64, device=device, generator=g)
        im = torch.randn(*shape, dtype=torch.float64, device=device, generator=g)
        return torch.complex(re, im)

    q, r = torch.linalg.qr(cnormal(n, n))
    d = torch.diagonal(r)
    u = q * (d / d.abs())
    del q, r
    a_vals = lo + (hi - lo) * torch.rand(n, dtype=torch.float64, device=device, generator=g)
    A = (u * a_vals.to(torch.complex128)) @ u.conj().T
    del u
    A = 0.5 * (A + A.conj().T)
    G = cnormal(n, n)
    B = 0.5 * (G + G.T)
    del G
    x = cnormal(n)
    x = x / torch.linalg.vector_norm(x)
    val = torch.tensor(0.0, dtype=torch.float64, device=device)
    for _ in range(200):
        y = B.conj().T @ (B @ x)
        val = torch.linalg.vector_norm(y)
        x = y / val
    target = 1.0 if bnorm == "one" else 0.9 * float(a_vals.min())
    B = B * (target / float(torch.sqrt(val)))
    dip = cnormal(n)
    return A, B, dip, torch.sort(a_vals, descending=True).values


def random_bse(n, seed, margin=1.0, kind="complex"):
    """The reference suite's generator (core.random_bse, core.py:245-278,
    restated): Hermitian A0 and symmetric B0 with entries in [-1, 1], A
    shifted by (|A0|_F + |B0|_F + margin) I, which makes both validation
    checks pass (the Frobenius norms bound the spectral norms)."""
    from .types import make_operator
    if n < 1:
        raise ValueError("n must be at least 1")
    if margin <= 0.0:
        raise ValueError("margin must be positive")
    rng = np.random.default_rng(seed)
    if kind == "complex":
        g = rng.uniform(-1.0, 1.0, (n, n)) + 1j * rng.uniform(-1.0, 1.0, (n, n))
        a0 = 0.5 * (g + g.conj().T)
        g2 = rng.uniform(-1.0, 1.0, (n, n)) + 1j * rng.uniform(-1.0, 1.0, (n, n))
        b0 = 0.5 * (g2 + g2.T)
    elif kind == "real":
        g = rng.uniform(-1.0, 1.0, (n, n))
        a0 = 0.5 * (g + g.T)
        g2 = rng.uniform(-1.0, 1.0, (n, n))
        b0 = 0.5 * (g2 + g2.T)
    else:
        raise ValueError(f"kind must be 'real' or 'complex', got {kind!r}")
    shift = np.linalg.norm(a0) + np.linalg.norm(b0) + margin
    return make_operator(a0 + shift * np.eye(n), b0, kind=kind)


def config_operator_any(idx, n=None, seed=None):
    """config_operator on the host for small n; the GPU generators (torch)
    for n >= 4096 when a device is present (the host QRs of cfg2-4 take
    minutes).  Returns numpy (A, B, dipole n-vector)."""
    c = CONFIGS[idx]
    n = c["n"] if n is None else n
    seed = idx if seed is None else seed
    try:
        import torch
        gpu = torch.cuda.is_available() and n >= 4096
    except ImportError:
        gpu = False
    if not gpu:
        a, b, d2n = config_operator(idx, n=n, seed=seed)
        return a, b, d2n[:n]
    if c["kind"] == "real":
        S, D, dip = torch_real_operator(n, seed=seed, spectrum=c["spectrum"], lo=c["lo"],
                                        hi=c["hi"])
        a = (0.5 * (S + D)).cpu().numpy()
        b = (0.5 * (S - D)).cpu().numpy()
        return a, b, dip.cpu().numpy()
    A, B, dip, _ = torch_complex_operator(n, seed=seed, lo=c["lo"], hi=c["hi"], bnorm=c["bnorm"])
    return A.cpu().numpy(), B.cpu().numpy(), dip.cpu().numpy()
