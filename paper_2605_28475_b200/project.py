"""Batched general projection on the GPU: the drop-in for ``basis.project``.

The reference projects a velocity-space function onto the basis by sampling it
on a (radial x polar x azimuthal) product grid (basis.py:262-299):

* radial: generalized Gauss-Laguerre in x = v^2/2 (weight x^{1/2} e^{-x}) of
  the requested order, v = sqrt(2x), weight sqrt(2) w e^{x} (:276-279);
* polar: Gauss-Legendre in cos(theta), n_t = max(l_max + 1, order) (:281);
* azimuth: periodic trapezoid, n_p = 2 n_t + 1 (:282);
* points in (v, t, p) order, p fastest (:284-290).

``project_points`` returns exactly those points, so a caller evaluates its f
wherever it likes (numpy on the host, torch on the device) and hands the
samples to ``Projector.project`` -- one ``bfq_project_samples`` launch for the
whole batch (csrc/bfq_project_samples.cu).  ``project(f, cfg, order)`` is the
single-cell drop-in with the reference's signature and error behaviour.

The quadrature rules are the reference's own algorithms (Golub-Welsch plus two
Newton passes, quadrature.py:38-128), restated in ``rbuild``; the polar factor
and the radial functions follow basis.py:112-173, :244-258.
"""

from __future__ import annotations

import ctypes
import math
from functools import lru_cache

import numpy as np
from scipy.special import lpmv

from . import _lib, rbuild
from .inputs import radial_basis
from .operator import CoefficientField


@lru_cache(maxsize=16)
def projection_grid(l_max: int, order: int):
    """(v, radial weight, cos_t, w_t, phi, w_p) of basis.project (basis.py:272-282)."""
    if order < 1:
        raise ValueError("radial quadrature order must be positive")
    x, w = rbuild._laguerre_rule(order, 0.5)
    v = np.sqrt(2.0 * x)
    r_w = math.sqrt(2.0) * w * np.exp(x)
    n_t = max(l_max + 1, order)
    n_p = 2 * n_t + 1
    cos_t, w_t = rbuild._legendre_rule(n_t)
    phi = 2.0 * np.pi * np.arange(n_p) / n_p
    w_p = np.full(n_p, 2.0 * np.pi / n_p)
    return v, r_w, cos_t, w_t, phi, w_p


def project_points(cfg, order: int) -> np.ndarray:
    """The (n_v n_t n_p, 3) sample points, in the reference's order (basis.py:284-290)."""
    v, _, cos_t, _, phi, _ = projection_grid(cfg.l_max, order)
    sin_t = np.sqrt(1.0 - cos_t**2)
    vx = v[:, None, None] * (sin_t[:, None] * np.cos(phi)[None, :])[None]
    vy = v[:, None, None] * (sin_t[:, None] * np.sin(phi)[None, :])[None]
    vz = v[:, None, None] * (cos_t[:, None] * np.ones_like(phi))[None]
    return np.stack([vx, vy, vz], axis=-1).reshape(-1, 3)


def projection_tables(cfg, order: int):
    """Host tables of bfq_projector_create: azimuthal weights x {1, cos, sin}
    [2L+1][n_p] (column 0: m = 0, 2m-1: sin |m| phi, 2m: cos m phi), polar factor
    x weight [(l,|m|)][n_t] with the real-harmonic sign (-1)^m sqrt2 for m > 0,
    radial function x radial weight [l][k][v]."""
    L, n_k = cfg.l_max, cfg.n_k
    v, r_w, cos_t, w_t, phi, w_p = projection_grid(L, order)
    phi_tab = np.empty((2 * L + 1, phi.size))
    phi_tab[0] = w_p
    for m in range(1, L + 1):
        phi_tab[2 * m - 1] = w_p * np.sin(m * phi)
        phi_tab[2 * m] = w_p * np.cos(m * phi)
    theta_tab = np.empty(((L + 1) * (L + 2) // 2, cos_t.size))
    for l in range(L + 1):
        for m in range(l + 1):
            norm = math.exp(0.5 * (math.log((2 * l + 1) / (4.0 * math.pi))
                                   + math.lgamma(l - m + 1.0) - math.lgamma(l + m + 1.0)))
            sign = 1.0 if m == 0 else (-1.0) ** m * math.sqrt(2.0)
            theta_tab[l * (l + 1) // 2 + m] = sign * norm * lpmv(m, l, cos_t) * w_t
    radial_tab = np.empty((L + 1, n_k, v.size))
    for l in range(L + 1):
        radial_tab[l] = radial_basis(n_k, l, v) * r_w
    return (np.ascontiguousarray(phi_tab), np.ascontiguousarray(theta_tab), np.ascontiguousarray(radial_tab),
            (v.size, cos_t.size, phi.size))


class Projector:
    """Device projector for one (cfg, order): ``project(samples)`` maps a batch of
    sampled distributions (B, n_points) or (B, n_v, n_t, n_p), fp64 CUDA, to
    coefficients (B, n_k, n_q)."""

    def __init__(self, cfg, order: int, device: int | None = None):
        import torch

        self.cfg, self.order = cfg, order
        self.device = torch.cuda.current_device() if device is None else int(device)
        phi_tab, theta_tab, radial_tab, (self.n_v, self.n_t, self.n_p) = projection_tables(cfg, order)
        self.n_points = self.n_v * self.n_t * self.n_p
        lib = _lib.lib()
        h = ctypes.c_void_p()
        f64p = ctypes.POINTER(ctypes.c_double)
        _lib.check(lib.bfq_projector_create(cfg.k_max, cfg.l_max, self.n_v, self.n_t, self.n_p,
                                            phi_tab.ctypes.data_as(f64p), theta_tab.ctypes.data_as(f64p),
                                            radial_tab.ctypes.data_as(f64p), self.device, ctypes.byref(h)))
        self._h = h
        fl, by = ctypes.c_double(), ctypes.c_double()
        _lib.check(lib.bfq_projector_work(h, ctypes.byref(fl), ctypes.byref(by)))
        self.flops_per_cell, self.bytes_per_cell = fl.value, by.value
        self.kernel = int(lib.bfq_projector_kernel(h))  # 1 general, 2 register-tiled, 3 mirror-folded

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            try:
                _lib.lib().bfq_projector_destroy(h)
            except Exception:  # pragma: no cover - interpreter shutdown
                pass
            self._h = None

    def project(self, samples, out=None):
        import torch

        if not (isinstance(samples, torch.Tensor) and samples.is_cuda and samples.dtype == torch.float64):
            raise ValueError("samples must be a float64 CUDA tensor")
        if samples.device.index != self.device:
            raise ValueError(f"samples live on cuda:{samples.device.index}, the projector on cuda:{self.device}")
        b = samples.shape[0] if samples.dim() > 0 else 0
        if samples.numel() != b * self.n_points or samples.dim() not in (2, 4):
            raise ValueError(f"samples must have shape (B, {self.n_points}) or (B, {self.n_v}, {self.n_t}, {self.n_p})")
        if not samples.is_contiguous():
            raise ValueError("samples must be C-contiguous")
        cfg = self.cfg
        if out is None:
            out = torch.empty((b, cfg.n_k, cfg.n_q), dtype=torch.float64, device=samples.device)
        elif out.shape != (b, cfg.n_k, cfg.n_q) or out.dtype != torch.float64 or not out.is_contiguous() \
                or out.device != samples.device:
            raise ValueError("out must be a contiguous float64 (B, n_k, n_q) tensor on the samples' device")
        with torch.cuda.device(self.device):
            st = torch.cuda.current_stream(self.device).cuda_stream
            _lib.check(_lib.lib().bfq_project_samples(self._h, ctypes.c_void_p(samples.data_ptr()),
                                                      ctypes.c_void_p(out.data_ptr()), b, ctypes.c_void_p(st)))
        return out


@lru_cache(maxsize=8)
def _projector(cfg_key, order: int, device: int):
    from .operator import SpectralConfig

    return Projector(SpectralConfig(*cfg_key), order, device)


def project(f, cfg, radial_quad_order: int) -> CoefficientField:
    """Drop-in for ``basis.project(f, cfg, radial_quad_order)`` (basis.py:262-299):
    f is called once with the (n_points, 3) points and returns its values; the
    quadrature runs on the GPU."""
    import torch

    if radial_quad_order < 1:
        raise ValueError("radial quadrature order must be positive")
    pts = project_points(cfg, radial_quad_order)
    fv = np.asarray(f(pts), dtype=float).reshape(1, -1)
    dev = torch.cuda.current_device()
    pj = _projector((cfg.k_max, cfg.l_max, cfg.gamma), radial_quad_order, dev)
    c = pj.project(torch.from_numpy(np.ascontiguousarray(fv)).to(torch.device("cuda", dev)))
    return CoefficientField(c[0].cpu().numpy(), cfg)
