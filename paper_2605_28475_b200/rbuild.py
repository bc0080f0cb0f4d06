"""GPU operator build: the reference's ``build_operator`` with the R-tensor
integrals on the B200.

Host side of ``include/bfr.h``.  The reference spends its whole build
(21 min on 8 cores at N=L=12, hours at N=L=16) in
``kinematic.assemble_r_tensor`` (kinematic.py:521-570); here the host only
prepares the small exact tables -- quadrature rules (quadrature.py:38-128),
Wigner 3-j symbols (angular.py:35-95), Laguerre monomial coefficients and
radial norms (basis.py:112-173), the channel list (angular.py:117-131) -- and
``bfr_assemble`` evaluates every grid, harmonic, radial function and channel
integral on the device.  There is no CPU fallback: without the CUDA library
the build raises.

Public API mirrors the reference:

* ``grid_sizes`` / ``check_grid``      -- quadrature.py:162-220
* ``assemble_r_tensor(cfg, grid, *, kernel_scale, threads)`` -- kinematic.py:521-570
* ``apply_conservation`` / ``apply_detailed_balance``        -- kinematic.py:580-620
* ``build_gaunt_coo(l_max)``           -- angular.py:252-288
* ``build_operator(cfg, pad_rad, pad_ang, *, grid, threads, conservation,
  detailed_balance, kernel_scale)``    -- contraction.py:158-177
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass, replace
from functools import lru_cache

import numpy as np
from scipy.linalg import eigh_tridiagonal

from . import _lib
from .operator import (
    ChannelTable,
    FactorizedOperator,
    GauntCOO,
    RTensor,
    SpectralConfig,
    q_index,
    slices_from_rows,
)

__all__ = [
    "GridSpec",
    "grid_baseline",
    "grid_sizes",
    "check_grid",
    "wigner3j",
    "enumerate_channels",
    "assemble_r_tensor",
    "apply_conservation",
    "apply_detailed_balance",
    "build_gaunt_coo",
    "build_operator",
    "last_stats",
    "register_with_reference",
]


# ------------------------------------------------------------------ grid
@dataclass(frozen=True)
class GridSpec:
    """Per-axis point counts of the 5D kinematic grid (quadrature.py:131-160)."""

    n_e: int
    n_rho1: int
    n_t1: int
    n_h2: int
    n_t2: int
    n_chi: int
    n_eps: int
    pad_rad: int
    pad_ang: int

    def as_tuple(self):
        return (self.n_e, self.n_rho1, self.n_t1, self.n_h2, self.n_t2, self.n_chi, self.n_eps,
                self.pad_rad, self.pad_ang)


def grid_baseline(k_max: int, l_max: int) -> GridSpec:
    """Exactness counts of the polynomial integrand (quadrature.py:162-173)."""
    if k_max < 0 or l_max < 0:
        raise ValueError("truncation limits must be non-negative")
    n_out = 4 * k_max + 3 * l_max + 4
    return GridSpec((6 * k_max + 3 * l_max + 9) // 4, n_out, k_max + (3 * l_max + 1) // 2 + 1, n_out,
                    3 * k_max + (3 * l_max) // 2 + 3, k_max + (l_max + 1) // 2 + 1, 2 * k_max + l_max + 1,
                    0, 0)


def grid_sizes(k_max: int, l_max: int, pad_rad: int = 16, pad_ang: int = 16) -> GridSpec:
    """Selective padding of the coupled kinematic axes (quadrature.py:176-196)."""
    if pad_rad < 0 or pad_ang < 0:
        raise ValueError("padding must be non-negative")
    b = grid_baseline(k_max, l_max)
    return GridSpec(b.n_e + pad_rad, b.n_rho1 + pad_rad, b.n_t1 + pad_ang, b.n_h2 + pad_ang,
                    b.n_t2 + pad_rad, b.n_chi, b.n_eps, pad_rad, pad_ang)


def check_grid(spec: GridSpec, k_max: int, l_max: int) -> None:
    """Raise ValueError if an axis is below the exactness baseline (quadrature.py:199-220)."""
    base = grid_baseline(k_max, l_max)
    for name in ("n_e", "n_rho1", "n_t1", "n_h2", "n_t2", "n_chi", "n_eps"):
        got, need = getattr(spec, name), getattr(base, name)
        if got < need:
            raise ValueError(f"grid axis {name}={got} below exactness baseline {need} "
                             f"for k_max={k_max}, l_max={l_max}")


# ------------------------------------------------------------------ rules
def _jacobi_rule(diag, offsq, mu0):
    """Golub-Welsch: eigenvalues of the Jacobi matrix, weights from the first
    eigenvector components (quadrature.py:38-51)."""
    if diag.size == 1:
        return diag.copy(), np.array([mu0])
    x, vec = eigh_tridiagonal(diag, np.sqrt(offsq[1:]))
    return x, mu0 * vec[0, :] ** 2


def _legendre_rule(n):
    """Gauss-Legendre on [-1,1] with two Newton passes (quadrature.py:63-80)."""
    if n < 1:
        raise ValueError(f"need at least one node, got n={n}")
    k = np.arange(n, dtype=float)
    off = np.zeros(n)
    off[1:] = k[1:] ** 2 / (4.0 * k[1:] ** 2 - 1.0)
    x, _ = _jacobi_rule(np.zeros(n), off, 2.0)
    if n == 1:
        return x, np.array([2.0])

    def pair(x):
        p0, p1 = np.ones_like(x), x.copy()
        for j in range(1, n):
            p1, p0 = ((2 * j + 1) * x * p1 - j * p0) / (j + 1), p1
        return p1, p0

    for _ in range(2):
        p, pm = pair(x)
        x = x - p / (n * (x * p - pm) / (x**2 - 1.0))
    p, pm = pair(x)
    dp = n * (x * p - pm) / (x**2 - 1.0)
    return x, 2.0 / ((1.0 - x**2) * dp**2)


def _legendre01(n):
    x, w = _legendre_rule(n)
    return 0.5 * (x + 1.0), 0.5 * w


def _laguerre_rule(n, a):
    """Generalised Gauss-Laguerre, weight x^a e^-x (quadrature.py:98-125)."""
    if n < 1:
        raise ValueError(f"need at least one node, got n={n}")
    if a <= -1.0:
        raise ValueError(f"generalized Laguerre weight requires a > -1, got a={a}")
    k = np.arange(n, dtype=float)
    off = np.zeros(n)
    off[1:] = k[1:] * (k[1:] + a)
    x, w = _jacobi_rule(2.0 * k + a + 1.0, off, math.gamma(a + 1.0))
    if n == 1:
        return x, w

    def pair(x):
        p0, p1 = np.ones_like(x), 1.0 + a - x
        for j in range(1, n):
            p1, p0 = ((2 * j + a + 1 - x) * p1 - (j + a) * p0) / (j + 1), p1
        return p1, p0

    for _ in range(2):
        p, pm = pair(x)
        x = x - p / ((n * p - (n + a) * pm) / x)
    _, pm = pair(x)
    lw = math.lgamma(n + a) - math.lgamma(n + 1.0) + np.log(x) - 2.0 * np.log(np.abs(pm))
    return x, np.exp(lw) / (n + a)


# ------------------------------------------------------------------ angular
@lru_cache(maxsize=None)
def _w3j_exact(l1, l2, l3, m1, m2, m3):
    f = math.factorial
    lo = max(0, l2 - l3 - m1, l1 - l3 + m2)
    hi = min(l1 + l2 - l3, l1 - m1, l2 + m2)
    num, den = 0, 1
    for t in range(lo, hi + 1):  # Racah single sum as one exact rational
        d = (f(t) * f(l3 - l2 + t + m1) * f(l3 - l1 + t - m2) * f(l1 + l2 - l3 - t)
             * f(l1 - t - m1) * f(l2 - t + m2))
        num = num * d + (-1) ** t * den
        den *= d
    if num == 0:
        return 0.0
    nn = f(l1 + l2 - l3) * f(l1 - l2 + l3) * f(-l1 + l2 + l3)
    for l, m in ((l1, m1), (l2, m2), (l3, m3)):
        nn *= f(l + m) * f(l - m)
    val = math.sqrt((num * num * nn) / (den * den * f(l1 + l2 + l3 + 1)))
    return (-1) ** (l1 - l2 - m3) * (1 if num > 0 else -1) * val


def wigner3j(l1, l2, l3, m1, m2, m3) -> float:
    """Wigner 3-j symbol, exact-integer Racah sum (angular.py:35-95).

    Evaluated on the same canonical column order / m sign as the reference so
    that equivalent requests share one correctly-rounded value."""
    l1, l2, l3, m1, m2, m3 = (int(v) for v in (l1, l2, l3, m1, m2, m3))
    if min(l1, l2, l3) < 0:
        raise ValueError("polar degrees must be non-negative")
    if abs(m1) > l1 or abs(m2) > l2 or abs(m3) > l3 or m1 + m2 + m3 != 0:
        return 0.0
    if l3 < abs(l1 - l2) or l3 > l1 + l2:
        return 0.0
    cols = [(l1, m1), (l2, m2), (l3, m3)]
    order = sorted(range(3), key=lambda i: cols[i])
    odd = (l1 + l2 + l3) % 2 == 1
    inversions = sum(1 for i in range(3) for j in range(i + 1, 3) if order[i] > order[j])
    sign = -1.0 if (inversions % 2 and odd) else 1.0
    cols = [cols[i] for i in order]
    ms = tuple(c[1] for c in cols)
    if tuple(-m for m in ms) < ms:
        ms = tuple(-m for m in ms)
        if odd:
            sign = -sign
    return sign * _w3j_exact(cols[0][0], cols[1][0], cols[2][0], *ms)


def enumerate_channels(l_max: int) -> ChannelTable:
    """Triangle + parity rule, lexicographic (angular.py:117-131)."""
    if l_max < 0:
        raise ValueError("l_max must be non-negative")
    trip = [(a, b, c) for a in range(l_max + 1) for b in range(l_max + 1) for c in range(l_max + 1)
            if abs(b - c) <= a <= b + c and (a + b + c) % 2 == 0]
    return ChannelTable.from_triplets(l_max, trip)


def _channel_scale(l1, l2, l3):
    lam = math.sqrt((2 * l1 + 1) * (2 * l2 + 1) * (2 * l3 + 1) / (4.0 * math.pi)) \
        * wigner3j(l1, l2, l3, 0, 0, 0)
    return 8.0 * math.pi**2 / lam


# ------------------------------------------------------------------ radial
def _radial_norm(k, l):
    return math.exp(0.5 * (1.5 * math.log(2.0 * math.pi) + math.lgamma(k + 1.0)
                           - (l + 0.5) * math.log(2.0) - math.lgamma(k + l + 1.5)))


def _mono(n_k, a):
    c = np.zeros((n_k, n_k))
    for k in range(n_k):
        for j in range(k + 1):
            lb = math.lgamma(k + a + 1.0) - math.lgamma(j + a + 1.0) - math.lgamma(k - j + 1.0)
            c[k, j] = (-1.0) ** j * math.exp(lb - math.lgamma(j + 1.0))
    return c


# ------------------------------------------------------------------ assembly
_LAST_STATS: dict = {}


def last_stats() -> dict:
    """Device timings / work of the most recent ``assemble_r_tensor`` call."""
    return dict(_LAST_STATS)


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def assemble_r_tensor(cfg: SpectralConfig, grid: GridSpec | None = None, *, kernel_scale: float = 1.0,
                      threads: int = 1, device: int | None = None, return_halves: bool = False):
    """Integrate the physical tensor for every channel on the GPU.

    Same result as kinematic.assemble_r_tensor (kinematic.py:521-570): gain +
    channel-swapped gain - both loss branches, slot-(2,3) symmetrised and
    channel-scaled, *before* the null-space corrections.  ``threads`` is
    accepted for signature compatibility (the device does the work).
    """
    del threads
    if device is None:  # the caller's current CUDA device, as torch sees it
        from .engine import _default_device

        device = _default_device()
    if grid is None:
        grid = grid_sizes(cfg.k_max, cfg.l_max)
    check_grid(grid, cfg.k_max, cfg.l_max)
    chans = enumerate_channels(cfg.l_max)
    n_k, L, n_t = cfg.n_k, cfg.l_max, chans.n_t
    trip = np.ascontiguousarray(chans.triplets, dtype=np.int32).reshape(n_t, 3)
    swap = np.array([chans.tau(l1, l3, l2) - 1 for (l1, l2, l3) in chans.triplets], dtype=np.int32)
    w3j = np.zeros((n_t, L + 1))
    for t, (l1, l2, l3) in enumerate(chans.triplets):
        for m in range(min(l1, l3) + 1):
            w3j[t, m] = wigner3j(l1, l2, l3, m, 0, -m)
    scale = np.array([_channel_scale(*t) for t in chans.triplets])
    e_x, e_w = _laguerre_rule(grid.n_e, 0.5 * cfg.gamma)
    chi_x, chi_w = _legendre_rule(grid.n_chi)
    eps_x = 2.0 * np.pi * np.arange(grid.n_eps) / grid.n_eps
    eps_w = np.full(grid.n_eps, 2.0 * np.pi / grid.n_eps)
    rules = [(_legendre01(grid.n_rho1), _legendre01(grid.n_t1)),
             (_legendre01(grid.n_h2), _legendre01(grid.n_t2))]
    mono = np.stack([_mono(n_k, l + 0.5) for l in range(L + 1)])
    norms = np.array([[_radial_norm(k, l) for k in range(n_k)] for l in range(L + 1)])

    keep = []  # arrays must outlive the call

    def f64p(a):
        a = _f64(a)
        keep.append(a)
        return a.ctypes.data_as(_lib._f64p)

    def i32p(a):
        a = np.ascontiguousarray(a, dtype=np.int32)
        keep.append(a)
        return a.ctypes.data_as(_lib._i32p)

    d = _lib.BfrDesc()
    d.k_max, d.l_max, d.gamma, d.kernel_scale = cfg.k_max, L, float(cfg.gamma), float(kernel_scale)
    d.n_t = n_t
    d.triplets, d.swap, d.w3j, d.chan_scale = i32p(trip), i32p(swap), f64p(w3j), f64p(scale)
    d.n_e, d.e_x, d.e_w = grid.n_e, f64p(e_x), f64p(e_w)
    d.n_chi, d.chi_x, d.chi_w = grid.n_chi, f64p(chi_x), f64p(chi_w)
    d.n_eps, d.eps_x, d.eps_w = grid.n_eps, f64p(eps_x), f64p(eps_w)
    for p, ((ox, ow), (tx, tw)) in enumerate(rules):
        d.n_outer[p], d.n_inner[p] = ox.size, tx.size
        d.outer_x[p], d.outer_w[p], d.inner_x[p], d.inner_w[p] = f64p(ox), f64p(ow), f64p(tx), f64p(tw)
    d.mono, d.norms = f64p(mono), f64p(norms)
    out = np.empty((n_k, n_k, n_k, n_t))
    halves = np.empty((3, n_t, n_k, n_k, n_k)) if return_halves else None
    st = _lib.BfrStats()
    _lib.check(_lib.lib().bfr_assemble(ctypes.byref(d), int(device), out.ctypes.data,
                                       halves.ctypes.data if halves is not None else None,
                                       ctypes.byref(st)))
    _LAST_STATS.clear()
    _LAST_STATS.update(ms_total=st.ms_total, ms_contract=st.ms_contract, contract_macs=st.contract_macs,
                       alg_macs=st.alg_macs, x_bytes=st.x_bytes,
                       n_points=(int(st.n_points[0]), int(st.n_points[1])), launches=int(st.launches))
    r = RTensor(out, chans, float(cfg.gamma), grid)
    if return_halves:
        return r, halves
    return r


def apply_conservation(r: RTensor) -> RTensor:
    """Zero the k1 rows that map onto mass/momentum (l1 <= 1, k1 = 0) and
    energy (l1 = 0, k1 = 1); idempotent (kinematic.py:580-600)."""
    vals = r.values.copy()
    worst = r.max_zeroed
    for t, (l1, _, _) in enumerate(r.channels.triplets):
        if l1 <= 1:
            worst = max(worst, float(np.max(np.abs(vals[0, :, :, t]))))
            vals[0, :, :, t] = 0.0
        if l1 == 0 and r.n_k > 1:
            worst = max(worst, float(np.max(np.abs(vals[1, :, :, t]))))
            vals[1, :, :, t] = 0.0
    return replace(r, values=vals, conservation_applied=True, max_zeroed=worst)


def apply_detailed_balance(r: RTensor) -> RTensor:
    """Zero the equilibrium input column of the isotropic channel (kinematic.py:603-620)."""
    vals = r.values.copy()
    t0 = r.channels.tau(0, 0, 0) - 1
    worst = max(r.max_zeroed, float(np.max(np.abs(vals[:, 0, 0, t0]))))
    vals[:, 0, 0, t0] = 0.0
    return replace(r, values=vals, detailed_balance_applied=True, max_zeroed=worst)


# ------------------------------------------------------------------ Gaunt table
ZERO_THRESHOLD = 1e-15  # angular.py:29-32


@lru_cache(maxsize=None)
def _c2r(l):
    """Complex -> real harmonic unitary, rows/cols m = -l..l (angular.py:134-157)."""
    u = np.zeros((2 * l + 1, 2 * l + 1), dtype=complex)
    s = 1.0 / math.sqrt(2.0)
    u[l, l] = 1.0
    for m in range(1, l + 1):
        cs = (-1.0) ** m
        u[l + m, l + m] = cs * s
        u[l + m, l - m] = s
        u[l - m, l + m] = -1j * cs * s
        u[l - m, l - m] = 1j * s
    return u


def _real_gaunt_block(l1, l2, l3):
    """Real Gaunt coefficients of one channel (angular.py:160-188)."""
    pref = math.sqrt((2 * l1 + 1) * (2 * l2 + 1) * (2 * l3 + 1) / (4.0 * math.pi)) \
        * wigner3j(l1, l2, l3, 0, 0, 0)
    t = np.zeros((2 * l1 + 1, 2 * l2 + 1, 2 * l3 + 1))
    if pref != 0.0:
        for m2 in range(-l2, l2 + 1):
            for m3 in range(-l3, l3 + 1):
                m1 = -(m2 + m3)
                if abs(m1) <= l1:
                    t[m1 + l1, m2 + l2, m3 + l3] = pref * wigner3j(l1, l2, l3, m1, m2, m3)
    b = np.tensordot(_c2r(l1), t.astype(complex), axes=(1, 0))
    b = np.tensordot(_c2r(l2), b, axes=(1, 1)).transpose(1, 0, 2)
    b = np.tensordot(b, _c2r(l3), axes=(2, 1))
    if not np.allclose(b.imag, 0.0, atol=1e-13):
        raise AssertionError("real Gaunt block has a non-negligible imaginary part")
    return b.real


def build_gaunt_coo(l_max: int) -> GauntCOO:
    """Sparse real-Gaunt routing table sorted by (tau, q1, q2, q3) (angular.py:252-288)."""
    chans = enumerate_channels(l_max)
    cols = [[], [], [], [], []]
    for t0, (l1, l2, l3) in enumerate(chans.triplets):
        blk = _real_gaunt_block(l1, l2, l3)
        for i1, i2, i3 in np.argwhere(np.abs(blk) >= ZERO_THRESHOLD):
            cols[0].append(q_index(l1, int(i1) - l1))
            cols[1].append(q_index(l2, int(i2) - l2))
            cols[2].append(q_index(l3, int(i3) - l3))
            cols[3].append(t0 + 1)
            cols[4].append(blk[i1, i2, i3])
    q1, q2, q3, tau = (np.array(c, dtype=np.int32) for c in cols[:4])
    g = np.array(cols[4], dtype=float)
    order = np.lexsort((q3, q2, q1, tau))
    q1, q2, q3, tau, g = q1[order], q2[order], q3[order], tau[order], g[order]
    n_q = (l_max + 1) ** 2
    starts, s_tau, s_q1 = slices_from_rows(tau, q1, n_q)
    return GauntCOO(l_max, n_q, chans, q1, q2, q3, tau, g, starts, s_tau, s_q1)


def build_operator(cfg: SpectralConfig, pad_rad: int = 16, pad_ang: int = 16, *,
                   grid: GridSpec | None = None, threads: int = 1, conservation: bool = True,
                   detailed_balance: bool = True, kernel_scale: float = 1.0,
                   device: int | None = None) -> FactorizedOperator:
    """Assemble the factorized operator with the null-space corrections
    (contraction.py:158-177), R integrals on the GPU."""
    if grid is None:
        grid = grid_sizes(cfg.k_max, cfg.l_max, pad_rad, pad_ang)
    r = assemble_r_tensor(cfg, grid, kernel_scale=kernel_scale, threads=threads, device=device)
    if conservation:
        r = apply_conservation(r)
    if detailed_balance:
        r = apply_detailed_balance(r)
    return FactorizedOperator(r, build_gaunt_coo(cfg.l_max), cfg)


def register_with_reference(kinematic_module=None, contraction_module=None) -> bool:
    """Route the reference's operator build through the GPU assembler.

    ``boltzfact.contraction.build_operator`` calls ``assemble_r_tensor`` by the
    name it imported from ``kinematic`` (contraction.py:22-25, :172), so both
    module attributes are replaced.  The returned ``RTensor`` carries the
    attributes the reference's ``apply_conservation`` / ``apply_detailed_balance``
    / ``FactorizedOperator`` / ``save_cache`` use (values, channels, gamma,
    grid.as_tuple(), flags, max_zeroed).  Returns False if the reference is not
    importable."""
    try:
        if kinematic_module is None:
            import boltzfact.kinematic as kinematic_module  # noqa: PLC0415
        if contraction_module is None:
            import boltzfact.contraction as contraction_module  # noqa: PLC0415
    except ImportError:
        return False
    kinematic_module.assemble_r_tensor = assemble_r_tensor
    contraction_module.assemble_r_tensor = assemble_r_tensor
    return True
