"""Seeded synthetic cells for the BASELINE configurations.

The benchmark has no public dataset; cells are drawn from the distributions
BASELINE.json names.  The reference builds a cell by quadrature projection of
a velocity-space function (basis.project, basis.py:262-299).  For a drifting
Maxwellian that projection has a closed angular form, which lets a whole
batch be generated in vectorised numpy on the GPU host:

    M_{u,T}(v) = (2 pi T)^{-3/2} exp(-|v-u|^2 / 2T),
    exp(v.u/T) = 4 pi sum_{lm} i_l(v|u|/T) Y_lm(v^) Y_lm(u^)      (addition theorem)
    c_{klm}    = (2/sqrt(pi)) e^{-|u|^2/2T} Y_lm(u^) sum_j w_j i_l(v_j |u|/T) phi_kl(v_j),
                 v_j = sqrt(2 T x_j), (x_j, w_j) generalized Gauss-Laguerre (alpha = 1/2),

with the reference's basis conventions: phi_kl(v) = N_kl v^l L_k^{(l+1/2)}(v^2/2)
(basis.py:105-135), orthonormal real harmonics built from the Condon-Shortley
Ferrers functions (basis.py:156-207), q = l^2 + l + m (0-based).
``tests/test_inputs.py`` pins it against the reference's ``project`` (golden
fixture + live check when the reference is importable).

Cells are generated in blocks of ``BLOCK`` with ``SeedSequence((seed, block))``
so every rank of a sharded run draws exactly its own cells of the global batch.
"""

from __future__ import annotations

import math

import numpy as np
from scipy.special import lpmv, roots_genlaguerre, spherical_in

BLOCK = 1024
INVARIANT_SLOTS = ((0, 0), (0, 1), (0, 2), (0, 3), (1, 0))  # (k, q) of mass/momentum/energy


def _radial_norms(n_k: int, l: int) -> np.ndarray:
    k = np.arange(n_k)
    log_n2 = (1.5 * math.log(2 * math.pi) + np.array([math.lgamma(x + 1.0) for x in k])
              - (l + 0.5) * math.log(2.0) - np.array([math.lgamma(x + l + 1.5) for x in k]))
    return np.exp(0.5 * log_n2)


def radial_basis(n_k: int, l: int, v: np.ndarray) -> np.ndarray:
    """phi_{k,l}(v) for k < n_k, shape (n_k,) + v.shape."""
    x = 0.5 * v * v
    a = l + 0.5
    lag = np.empty((n_k,) + v.shape)
    lag[0] = 1.0
    if n_k > 1:
        lag[1] = 1.0 + a - x
    for k in range(1, n_k - 1):
        lag[k + 1] = ((2 * k + a + 1 - x) * lag[k] - (k + a) * lag[k - 1]) / (k + 1)
    return _radial_norms(n_k, l).reshape((n_k,) + (1,) * v.ndim) * v**l * lag


def real_harmonics(l_max: int, dirs: np.ndarray) -> np.ndarray:
    """Y[..., q] for unit vectors dirs (..., 3), q = l^2 + l + m."""
    cos_t = np.clip(dirs[..., 2], -1.0, 1.0)
    phi = np.arctan2(dirs[..., 1], dirs[..., 0])
    out = np.empty(dirs.shape[:-1] + ((l_max + 1) ** 2,))
    for l in range(l_max + 1):
        for m in range(l + 1):
            norm = math.exp(0.5 * (math.log((2 * l + 1) / (4 * math.pi))
                                   + math.lgamma(l - m + 1.0) - math.lgamma(l + m + 1.0)))
            theta = norm * lpmv(m, l, cos_t)
            if m == 0:
                out[..., l * l + l] = theta
            else:
                s = math.sqrt(2.0) * (-1.0) ** m
                out[..., l * l + l + m] = s * theta * np.cos(m * phi)
                out[..., l * l + l - m] = s * theta * np.sin(m * phi)
    return out


def project_maxwellians(n_k: int, l_max: int, u: np.ndarray, temp: np.ndarray,
                        order: int = 96) -> np.ndarray:
    """Coefficients (B, n_k, n_q) of drifting Maxwellians M_{u_i, T_i}."""
    u = np.atleast_2d(np.asarray(u, dtype=float))
    temp = np.broadcast_to(np.asarray(temp, dtype=float), (u.shape[0],))
    b = u.shape[0]
    speed = np.linalg.norm(u, axis=1)
    dirs = np.where(speed[:, None] > 0, u / np.where(speed > 0, speed, 1.0)[:, None], [0.0, 0.0, 1.0])
    ylm = real_harmonics(l_max, dirs)  # (B, n_q)
    x, w = roots_genlaguerre(order, 0.5)
    v = np.sqrt(2.0 * temp[:, None] * x[None, :])  # (B, J)
    arg = v * (speed / temp)[:, None]
    pref = (2.0 / math.sqrt(math.pi)) * np.exp(-0.5 * speed * speed / temp)  # (B,)
    out = np.zeros((b, n_k, (l_max + 1) ** 2))
    for l in range(l_max + 1):
        rad = radial_basis(n_k, l, v)  # (n_k, B, J)
        bes = spherical_in(l, arg)  # (B, J)
        radial = np.einsum("kbj,bj,j->bk", rad, bes, w)  # (B, n_k)
        q = slice(l * l, (l + 1) * (l + 1))
        out[:, :, q] = (pref[:, None] * radial)[:, :, None] * ylm[:, None, q]
    return out


def noise_sigma(n_k: int, l_max: int) -> np.ndarray:
    """sigma_{k,l} = 1e-2 exp(-(k+l)/2) on the (n_k, n_q) grid (BASELINE.json configs)."""
    k = np.arange(n_k)[:, None]
    l = np.floor(np.sqrt(np.arange((l_max + 1) ** 2))).astype(int)[None, :]
    return 1e-2 * np.exp(-0.5 * (k + l))


def _zero_invariants(c: np.ndarray) -> None:
    for k, q in INVARIANT_SLOTS:
        if k < c.shape[-2] and q < c.shape[-1]:
            c[..., k, q] = 0.0


def _blocks(n_cells: int, start: int):
    first = start // BLOCK
    last = (start + n_cells + BLOCK - 1) // BLOCK
    for blk in range(first, last):
        lo = max(start, blk * BLOCK)
        hi = min(start + n_cells, (blk + 1) * BLOCK)
        yield blk, lo - blk * BLOCK, hi - blk * BLOCK, lo - start


def perturbed_maxwellians(n_k: int, l_max: int, n_cells: int, seed: int, start: int = 0) -> np.ndarray:
    """Configs 2-4: u ~ U(-0.3,0.3)^3, T ~ U(0.8,1.2), c = P[M_{u,T}] + N(0, sigma)
    with the noise zeroed on the five invariant slots."""
    out = np.empty((n_cells, n_k, (l_max + 1) ** 2))
    sig = noise_sigma(n_k, l_max)
    for blk, lo, hi, dst in _blocks(n_cells, start):
        rng = np.random.default_rng(np.random.SeedSequence((seed, blk)))
        u = rng.uniform(-0.3, 0.3, (BLOCK, 3))
        t = rng.uniform(0.8, 1.2, BLOCK)
        noise = rng.normal(size=(BLOCK, n_k, (l_max + 1) ** 2)) * sig
        _zero_invariants(noise)
        c = project_maxwellians(n_k, l_max, u[lo:hi], t[lo:hi]) + noise[lo:hi]
        out[dst:dst + hi - lo] = c
    return out


def maxwell_config1(n_k: int, l_max: int, seed: int, n_cells: int = 1) -> np.ndarray:
    """Config 1: c = N(0, sigma) everywhere, then c_000 = 1 and momentum/energy
    coefficients at their Maxwellian values (0)."""
    rng = np.random.default_rng(seed)
    c = rng.normal(size=(n_cells, n_k, (l_max + 1) ** 2)) * noise_sigma(n_k, l_max)
    _zero_invariants(c)
    c[:, 0, 0] = 1.0
    return c


def bimodal(n_k: int, l_max: int, n_cells: int, seed: int, start: int = 0) -> np.ndarray:
    """Config 5: f = 1/2 M_{+u n, 1} + 1/2 M_{-u n, 1}, u ~ U(0.5,1.5), n uniform on S^2."""
    out = np.empty((n_cells, n_k, (l_max + 1) ** 2))
    for blk, lo, hi, dst in _blocks(n_cells, start):
        rng = np.random.default_rng(np.random.SeedSequence((seed, blk)))
        u = rng.uniform(0.5, 1.5, BLOCK)
        n = rng.normal(size=(BLOCK, 3))
        n /= np.linalg.norm(n, axis=1, keepdims=True)
        d = (u[:, None] * n)[lo:hi]
        ones = np.ones(hi - lo)
        out[dst:dst + hi - lo] = 0.5 * (project_maxwellians(n_k, l_max, d, ones)
                                        + project_maxwellians(n_k, l_max, -d, ones))
    return out


def uniform_fields(n_k: int, l_max: int, n_cells: int, seed: int) -> np.ndarray:
    """The reference tests' random field: U(-1,1) with c_000 = 1 (test_contraction.py:20-24)."""
    rng = np.random.default_rng(seed)
    c = rng.uniform(-1.0, 1.0, (n_cells, n_k, (l_max + 1) ** 2))
    c[:, 0, 0] = 1.0
    return c


# ------------------------------------------------------------------ on the GPU
def project_maxwellians_device(n_k: int, l_max: int, u, temp, noise=None, order: int = 96, out=None):
    """``project_maxwellians`` on the device (bfq_project_maxwellians): u (B, 3),
    temp (B,) and the optional additive noise (B, n_k, n_q) are float64 CUDA
    tensors; returns the (B, n_k, n_q) CUDA tensor.  Same closed form and rule."""
    import ctypes

    import torch

    from . import _lib

    b = u.shape[0]
    if out is None:
        out = torch.empty((b, n_k, (l_max + 1) ** 2), dtype=torch.float64, device=u.device)
    for t, shape in ((u, (b, 3)), (temp, (b,)), (out, (b, n_k, (l_max + 1) ** 2))):
        if tuple(t.shape) != shape or t.dtype != torch.float64 or not t.is_cuda or not t.is_contiguous():
            raise ValueError(f"expected a contiguous float64 CUDA tensor of shape {shape}")
    if noise is not None and (tuple(noise.shape) != tuple(out.shape) or not noise.is_cuda
                              or noise.dtype != torch.float64 or not noise.is_contiguous()):
        raise ValueError("noise must match the output tensor")
    x, w = roots_genlaguerre(order, 0.5)
    x, w = np.ascontiguousarray(x), np.ascontiguousarray(w)
    stream = torch.cuda.current_stream(u.device).cuda_stream
    _lib.check(_lib.lib().bfq_project_maxwellians(
        n_k - 1, l_max, x.ctypes.data_as(_lib._f64p), w.ctypes.data_as(_lib._f64p), order,
        u.data_ptr(), temp.data_ptr(), noise.data_ptr() if noise is not None else None, out.data_ptr(),
        b, stream))
    return out


def perturbed_maxwellians_device(n_k: int, l_max: int, n_cells: int, seed: int, start: int = 0, device=0):
    """``perturbed_maxwellians`` with the projection on the GPU: the same seeded
    draws (u, T, noise per 1024-cell block), so the cells agree with the host
    generator to rounding.  Returns a float64 CUDA tensor."""
    import torch

    n_q = (l_max + 1) ** 2
    sig = noise_sigma(n_k, l_max)
    us, ts, ns = [], [], []
    for blk, lo, hi, _ in _blocks(n_cells, start):
        rng = np.random.default_rng(np.random.SeedSequence((seed, blk)))
        u = rng.uniform(-0.3, 0.3, (BLOCK, 3))
        t = rng.uniform(0.8, 1.2, BLOCK)
        noise = rng.normal(size=(BLOCK, n_k, n_q)) * sig
        _zero_invariants(noise)
        us.append(u[lo:hi])
        ts.append(t[lo:hi])
        ns.append(noise[lo:hi])
    dev = torch.device("cuda", device) if isinstance(device, int) else torch.device(device)
    to = lambda a: torch.from_numpy(np.ascontiguousarray(np.concatenate(a))).to(dev)  # noqa: E731
    return project_maxwellians_device(n_k, l_max, to(us), to(ts), noise=to(ns))


def bimodal_device(n_k: int, l_max: int, n_cells: int, seed: int, start: int = 0, device=0):
    """``bimodal`` (config 5) with the projection on the GPU."""
    import torch

    ds = []
    for blk, lo, hi, _ in _blocks(n_cells, start):
        rng = np.random.default_rng(np.random.SeedSequence((seed, blk)))
        u = rng.uniform(0.5, 1.5, BLOCK)
        n = rng.normal(size=(BLOCK, 3))
        n /= np.linalg.norm(n, axis=1, keepdims=True)
        ds.append((u[:, None] * n)[lo:hi])
    dev = torch.device("cuda", device) if isinstance(device, int) else torch.device(device)
    d = torch.from_numpy(np.ascontiguousarray(np.concatenate(ds))).to(dev)
    ones = torch.ones(d.shape[0], dtype=torch.float64, device=dev)
    a = project_maxwellians_device(n_k, l_max, d.contiguous(), ones)
    b = project_maxwellians_device(n_k, l_max, (-d).contiguous(), ones)
    return 0.5 * (a + b)
