"""CPU oracle for the R-tensor assembly -- TEST INFRASTRUCTURE ONLY.

Only ``tests/`` and ``bench.py``'s reference leg may import this module, and
only as the checker / the timed CPU port.  The product path
(``paper_2605_28475_b200.rbuild``) never calls it.

A numpy restatement of the reference's kinematic assembly
(``/root/reference/pkg/src/boltzfact/kinematic.py``), written for clarity,
not speed:

* quadrature rules -- quadrature.py:38-128 (Golub-Welsch + two Newton passes,
  weights from the derivative identities), grid sizes quadrature.py:162-196;
* Wigner 3-j -- angular.py:35-95 (Racah single sum over exact integers);
* radial functions / Laguerre monomials / polar harmonics --
  basis.py:112-141, 155-193;
* per-patch Duffy geometry -- kinematic.py:322-380;
* half-plane gain / loss integrals of one channel -- kinematic.py:408-510;
* full-plane combination, slot symmetrisation and channel scale --
  kinematic.py:513-570;
* null-space corrections -- kinematic.py:594-620.

Parity of this restatement is pinned by ``tests/test_rbuild.py``
against the R tensors of the reference-built operator caches in
``operators/`` (``boltzfact build``; the cache stores R after the
corrections).
"""

from __future__ import annotations

import math
from functools import lru_cache

import numpy as np
from scipy.linalg import eigh_tridiagonal
from scipy.special import lpmv


# ----------------------------------------------------------------- rules
def _gw(alpha, beta, mu0):
    if alpha.size == 1:
        return alpha.copy(), np.array([mu0])
    vals, vecs = eigh_tridiagonal(alpha, np.sqrt(beta[1:]))
    return vals, mu0 * vecs[0, :] ** 2


def _leg_pair(n, x):
    p0, p1 = np.ones_like(x), x.copy()
    for k in range(1, n):
        p1, p0 = ((2 * k + 1) * x * p1 - k * p0) / (k + 1), p1
    return p1, p0


def gauss_legendre(n):
    """quadrature.py:60-80."""
    k = np.arange(n, dtype=float)
    beta = np.zeros(n)
    beta[1:] = k[1:] ** 2 / (4.0 * k[1:] ** 2 - 1.0)
    x, _ = _gw(np.zeros(n), beta, 2.0)
    if n == 1:
        return x, np.array([2.0])
    for _ in range(2):
        p, pm = _leg_pair(n, x)
        x = x - p / (n * (x * p - pm) / (x * x - 1.0))
    p, pm = _leg_pair(n, x)
    dp = n * (x * p - pm) / (x * x - 1.0)
    return x, 2.0 / ((1.0 - x * x) * dp * dp)


def gauss_legendre_01(n):
    x, w = gauss_legendre(n)
    return 0.5 * (x + 1.0), 0.5 * w


def _lag_pair(n, a, x):
    p0, p1 = np.ones_like(x), 1.0 + a - x
    for k in range(1, n):
        p1, p0 = ((2 * k + a + 1 - x) * p1 - (k + a) * p0) / (k + 1), p1
    return p1, p0


def gauss_laguerre_gen(n, a):
    """quadrature.py:98-125."""
    k = np.arange(n, dtype=float)
    beta = np.zeros(n)
    beta[1:] = k[1:] * (k[1:] + a)
    x, w = _gw(2.0 * k + a + 1.0, beta, math.gamma(a + 1.0))
    if n == 1:
        return x, w
    for _ in range(2):
        p, pm = _lag_pair(n, a, x)
        x = x - p / ((n * p - (n + a) * pm) / x)
    _, pm = _lag_pair(n, a, x)
    lw = math.lgamma(n + a) - math.lgamma(n + 1.0) + np.log(x) - 2.0 * np.log(np.abs(pm))
    return x, np.exp(lw) / (n + a)


def grid_sizes(k_max, l_max, pad_rad=16, pad_ang=16):
    """quadrature.py:162-196 -> (n_e, n_rho1, n_t1, n_h2, n_t2, n_chi, n_eps)."""
    n_e = (6 * k_max + 3 * l_max + 9) // 4
    n_out = 4 * k_max + 3 * l_max + 4
    n_t1 = k_max + (3 * l_max + 1) // 2 + 1
    n_t2 = 3 * k_max + (3 * l_max) // 2 + 3
    n_chi = k_max + (l_max + 1) // 2 + 1
    n_eps = 2 * k_max + l_max + 1
    return (n_e + pad_rad, n_out + pad_rad, n_t1 + pad_ang, n_out + pad_ang, n_t2 + pad_rad,
            n_chi, n_eps)


# ----------------------------------------------------------------- angular
@lru_cache(maxsize=None)
def wigner3j(l1, l2, l3, m1, m2, m3):
    """Racah single-sum formula in exact integers (angular.py:35-61)."""
    if m1 + m2 + m3 != 0 or abs(m1) > l1 or abs(m2) > l2 or abs(m3) > l3:
        return 0.0
    if l3 < abs(l1 - l2) or l3 > l1 + l2:
        return 0.0
    f = math.factorial
    t0 = max(0, l2 - l3 - m1, l1 - l3 + m2)
    t1 = min(l1 + l2 - l3, l1 - m1, l2 + m2)
    num, den = 0, 1
    for t in range(t0, t1 + 1):
        d = (f(t) * f(l3 - l2 + t + m1) * f(l3 - l1 + t - m2) * f(l1 + l2 - l3 - t)
             * f(l1 - t - m1) * f(l2 - t + m2))
        num = num * d + (-1) ** t * den
        den *= d
    if num == 0:
        return 0.0
    nn = f(l1 + l2 - l3) * f(l1 - l2 + l3) * f(-l1 + l2 + l3)
    for l, m in ((l1, m1), (l2, m2), (l3, m3)):
        nn *= f(l + m) * f(l - m)
    sq = (num * num * nn) / (den * den * f(l1 + l2 + l3 + 1))
    return (-1) ** (l1 - l2 - m3) * (1 if num > 0 else -1) * math.sqrt(sq)


def channels(l_max):
    """angular.py:117-131: triangle + parity, lexicographic."""
    return [(a, b, c) for a in range(l_max + 1) for b in range(l_max + 1) for c in range(l_max + 1)
            if abs(b - c) <= a <= b + c and (a + b + c) % 2 == 0]


def sph_theta(l, m, x):
    """basis.py:176-193: N_lm P_l^m(x), Condon-Shortley phase."""
    n = math.exp(0.5 * (math.log((2 * l + 1) / (4 * math.pi)) + math.lgamma(l - m + 1.0)
                        - math.lgamma(l + m + 1.0)))
    return n * lpmv(m, l, x)


def zonal(l):
    return math.sqrt((2 * l + 1) / (4.0 * math.pi))


# ----------------------------------------------------------------- radial
def radial_norm(k, l):
    return math.exp(0.5 * (1.5 * math.log(2 * math.pi) + math.lgamma(k + 1.0)
                           - (l + 0.5) * math.log(2.0) - math.lgamma(k + l + 1.5)))


def radial_all(l, v, n_k):
    """basis.py:123-141: phi_{k,l}(v), k < n_k."""
    x = 0.5 * v * v
    a = l + 0.5
    lag = np.empty((n_k,) + v.shape)
    lag[0] = 1.0
    if n_k > 1:
        lag[1] = 1.0 + a - x
    for k in range(1, n_k - 1):
        lag[k + 1] = ((2 * k + a + 1 - x) * lag[k] - (k + a) * lag[k - 1]) / (k + 1)
    nrm = np.array([radial_norm(k, l) for k in range(n_k)]).reshape((n_k,) + (1,) * v.ndim)
    return nrm * v**l * lag


def mono_coeffs(n_k, a):
    """basis.py:155-173: L_k^(a)(x) = sum_j C[k,j] x^j."""
    c = np.zeros((n_k, n_k))
    for k in range(n_k):
        for j in range(k + 1):
            lb = math.lgamma(k + a + 1.0) - math.lgamma(j + a + 1.0) - math.lgamma(k - j + 1.0)
            c[k, j] = (-1.0) ** j * math.exp(lb - math.lgamma(j + 1.0))
    return c


# ----------------------------------------------------------------- geometry
class Patch:
    """kinematic.py:322-380: one Duffy patch on its tensor grid."""

    def __init__(self, patch, outer, trule, chi, eps):
        self.patch = patch
        (xo, wo), (xt, wt) = outer, trule
        self.wo, self.wt = wo, wt
        self.w_chi = chi[1]
        self.w_eps = eps[1]
        x, t = xo[:, None], xt[None, :]
        if patch == 1:
            rho = np.broadcast_to(x, (x.size, t.size)).copy()
            h = x * t
            duffy = rho**2 * t
        else:
            h = np.broadcast_to(x, (x.size, t.size)).copy()
            rho = x * t
            duffy = np.broadcast_to(x, (x.size, t.size)) ** 2
        self.rho, self.h = rho, h
        self.cos_b = 1.0 - 2.0 * h**2
        sin_b = 2.0 * h * np.sqrt(np.clip(1.0 - h**2, 0.0, None))
        self.v0, self.w0 = 1.0 + rho, 1.0 - rho
        self.u0 = 2.0 * np.sqrt(rho**2 + (1.0 - rho**2) * h**2)
        self.f_geo = 4.0 * (2.0 * math.pi) ** -3 * duffy * (1.0 - rho**2) ** 2
        cx = 0.5 * self.w0 * sin_b
        cz = 0.5 * (self.v0 + self.w0 * self.cos_b)
        su = np.where(self.u0 > 0, self.u0, 1.0)
        uhx = -self.w0 * sin_b / su
        uhz = (self.v0 - self.w0 * self.cos_b) / su
        n1 = np.abs(uhx)
        deg = n1 < 1e-14
        sn = np.where(deg, 1.0, n1)
        e1x = np.where(deg, 1.0, -uhz * uhx / sn)
        e1z = np.where(deg, 0.0, uhx * uhx / sn)
        e2y = uhz * e1x - uhx * e1z
        cc = chi[0][:, None, None, None]
        sc = np.sqrt(np.clip(1.0 - cc**2, 0.0, None))
        ce = np.cos(eps[0])[None, :, None, None]
        se = np.sin(eps[0])[None, :, None, None]
        hu = 0.5 * self.u0[None, None]
        vx = cx[None, None] + hu * (cc * uhx[None, None] + sc * ce * e1x[None, None])
        vy = hu * sc * se * e2y[None, None]
        vz = cz[None, None] + hu * (cc * uhz[None, None] + sc * ce * e1z[None, None])
        self.vps = np.sqrt(vx**2 + vy**2 + vz**2)
        safe = np.where(self.vps > 0, self.vps, 1.0)
        self.cos_tp = np.clip(np.where(self.vps > 0, vz / safe, 1.0), -1.0, 1.0)
        phi = np.arctan2(vy, vx)
        self.cos_m = [np.ones_like(phi), np.cos(phi)]

    def cos_m_phi(self, m):
        while len(self.cos_m) <= m:
            k = len(self.cos_m)
            self.cos_m.append(2.0 * self.cos_m[1] * self.cos_m[k - 1] - self.cos_m[k - 2])
        return self.cos_m[m]


class Assembly:
    """kinematic.py:383-406 context + :408-510 half-plane integrals.

    ``precision="ld"`` evaluates the gain integrand from the m-sum through the
    monomial radial expansion (kinematic.py:427-471) in numpy long double
    (64-bit mantissa) -- a higher-precision restatement used to measure the
    reference's own fp64 rounding there (tests/precision/)."""

    def __init__(self, k_max, l_max, gamma, grid, kernel_scale=1.0, precision="f64"):
        self.precision = precision
        n_e, n_r1, n_t1, n_h2, n_t2, n_chi, n_eps = grid[:7]
        self.n_k, self.l_max, self.gamma, self.ks = k_max + 1, l_max, gamma, kernel_scale
        self.eta, self.w_e = gauss_laguerre_gen(n_e, 0.5 * gamma)
        chi = gauss_legendre(n_chi)
        eps = (2.0 * np.pi * np.arange(n_eps) / n_eps, np.full(n_eps, 2.0 * np.pi / n_eps))
        self.patches = [Patch(1, gauss_legendre_01(n_r1), gauss_legendre_01(n_t1), chi, eps),
                        Patch(2, gauss_legendre_01(n_h2), gauss_legendre_01(n_t2), chi, eps)]
        self.eta_pow = np.vstack([self.eta**j for j in range(self.n_k)])
        self.mono = {l: mono_coeffs(self.n_k, l + 0.5) for l in range(l_max + 1)}
        self.norms = {l: np.array([radial_norm(k, l) for k in range(self.n_k)])
                      for l in range(l_max + 1)}

    def _radial(self, geo, l, which):
        base = geo.v0 if which == "v" else geo.w0
        if geo.patch == 1:
            sp = np.sqrt(self.eta)[:, None] * base[:, 0][None, :]
        else:
            sp = np.sqrt(self.eta)[:, None, None] * base[None, :, :]
        return radial_all(l, sp, self.n_k)

    def patch_half(self, geo, l1, l2, l3):
        n_k, eta = self.n_k, self.eta
        if self.precision == "ld":
            return self._patch_half_ld(geo, l1, l2, l3)
        p_gain = np.zeros_like(geo.vps)
        for m in range(min(l1, l3) + 1):
            w3 = wigner3j(l1, l2, l3, m, 0, -m)
            if w3 == 0.0:
                continue
            b = (1.0 if m == 0 else 2.0) * (-1.0) ** m * w3 * sph_theta(l3, m, geo.cos_b)
            p_gain = p_gain + b[None, None] * (sph_theta(l1, m, geo.cos_tp) * geo.cos_m_phi(m))
        p_gain *= zonal(l2)
        p_loss = zonal(l1) * zonal(l2) * wigner3j(l1, l2, l3, 0, 0, 0) * sph_theta(l3, 0, geo.cos_b)
        kern = self.ks * geo.u0**self.gamma / (4.0 * math.pi)
        pw = geo.vps**l1 if l1 > 0 else np.ones_like(geo.vps)
        step = 0.5 * geo.vps**2
        gs = np.empty((n_k,) + geo.u0.shape)
        for j in range(n_k):
            if j > 0:
                pw = pw * step
            s = np.tensordot(pw * p_gain, geo.w_eps, axes=(1, 0))
            gs[j] = np.tensordot(s, geo.w_chi, axes=(0, 0)) * kern
        pref = self.norms[l1][:, None] * eta ** (0.5 * l1)
        core = np.einsum("kj,jE,jot->kEot", self.mono[l1], self.eta_pow, gs) * pref[:, :, None, None]
        r = {(l, w): self._radial(geo, l, w) for l in {l1, l2, l3} for w in "vw"}
        lk = (geo.w_chi.sum() * 2.0 * math.pi) * kern * p_loss
        if geo.patch == 1:
            rho1 = geo.rho[:, 0]
            env = self.w_e[:, None] * eta[:, None] ** 2 * np.exp(-eta[:, None] * rho1[None] ** 2) \
                * geo.wo[None, :]
            theta = np.tensordot(core * geo.f_geo[None, None], geo.wt, axes=(3, 0))
            gain = np.einsum("kEo,aEo,bEo,Eo->kab", theta, r[l2, "v"], r[l3, "w"], env)
            lenv = env * np.tensordot(geo.f_geo * lk, geo.wt, axes=(1, 0))
            lf = np.einsum("kEo,aEo,bEo,Eo->kab", r[l1, "v"], r[l2, "v"], r[l3, "w"], lenv)
            ls = np.einsum("kEo,aEo,bEo,Eo->kab", r[l1, "w"], r[l2, "w"], r[l3, "v"], lenv)
            return gain, lf, ls
        env = self.w_e[:, None, None] * eta[:, None, None] ** 2 \
            * np.exp(-eta[:, None, None] * geo.rho[None] ** 2) \
            * (geo.wo[:, None] * geo.wt[None, :] * geo.f_geo)[None]
        gain = np.einsum("kEot,aEot,bEot,Eot->kab", core, r[l2, "v"], r[l3, "w"], env)
        lenv = env * lk[None]
        lf = np.einsum("kEot,aEot,bEot,Eot->kab", r[l1, "v"], r[l2, "v"], r[l3, "w"], lenv)
        ls = np.einsum("kEot,aEot,bEot,Eot->kab", r[l1, "w"], r[l2, "w"], r[l3, "v"], lenv)
        return gain, lf, ls

    def _patch_half_ld(self, geo, l1, l2, l3):
        LD = np.longdouble
        n_k, eta = self.n_k, self.eta
        p_gain = np.zeros(geo.vps.shape, dtype=LD)
        for m in range(min(l1, l3) + 1):
            w3 = wigner3j(l1, l2, l3, m, 0, -m)
            if w3 == 0.0:
                continue
            b = (1.0 if m == 0 else 2.0) * (-1.0) ** m * w3 * sph_theta(l3, m, geo.cos_b)
            y = sph_theta(l1, m, geo.cos_tp) * geo.cos_m_phi(m)
            p_gain = p_gain + b[None, None].astype(LD) * y.astype(LD)
        p_gain *= LD(zonal(l2))
        vps = geo.vps.astype(LD)
        kern = (self.ks * geo.u0**self.gamma / (4.0 * math.pi)).astype(LD)
        pw, step = vps**l1, LD(0.5) * vps**2
        gs = np.empty((n_k,) + geo.u0.shape, dtype=LD)
        for j in range(n_k):
            if j > 0:
                pw = pw * step
            s = np.einsum("cest,e->cst", pw * p_gain, geo.w_eps.astype(LD))
            gs[j] = np.einsum("cst,c->st", s, geo.w_chi.astype(LD)) * kern
        pref = (self.norms[l1][:, None] * eta ** (0.5 * l1)).astype(LD)
        core = np.einsum("kj,jE,jot->kEot", self.mono[l1].astype(LD), self.eta_pow.astype(LD), gs)
        core = (core * pref[:, :, None, None]).astype(np.float64)
        self.precision = "f64"
        try:
            _, lf, ls = self.patch_half(geo, l1, l2, l3)
        finally:
            self.precision = "ld"
        r2v, r3w = self._radial(geo, l2, "v"), self._radial(geo, l3, "w")
        if geo.patch == 1:
            env = self.w_e[:, None] * eta[:, None] ** 2 * np.exp(-eta[:, None] * geo.rho[:, 0][None] ** 2) \
                * geo.wo[None, :]
            theta = np.tensordot(core * geo.f_geo[None, None], geo.wt, axes=(3, 0))
            return np.einsum("kEo,aEo,bEo,Eo->kab", theta, r2v, r3w, env), lf, ls
        env = self.w_e[:, None, None] * eta[:, None, None] ** 2 \
            * np.exp(-eta[:, None, None] * geo.rho[None] ** 2) \
            * (geo.wo[:, None] * geo.wt[None, :] * geo.f_geo)[None]
        return np.einsum("kEot,aEot,bEot,Eot->kab", core, r2v, r3w, env), lf, ls

    def channel_half(self, l1, l2, l3):
        """kinematic.py:390-406: both patches."""
        out = [np.zeros((self.n_k,) * 3) for _ in range(3)]
        for geo in self.patches:
            for acc, part in zip(out, self.patch_half(geo, l1, l2, l3)):
                acc += part
        return out


def channel_scale(l1, l2, l3):
    lam = math.sqrt((2 * l1 + 1) * (2 * l2 + 1) * (2 * l3 + 1) / (4 * math.pi)) \
        * wigner3j(l1, l2, l3, 0, 0, 0)
    return 8.0 * math.pi**2 / lam


def assemble_r(k_max, l_max, gamma, grid=None, kernel_scale=1.0, conservation=True,
               detailed_balance=True, only=None, precision="f64"):
    """kinematic.py:521-570 + 594-620 -> R (n_k, n_k, n_k, N_T).

    ``only``: optional list of 0-based channel indices; the others stay NaN
    (for spot checks at sizes where the full assembly is too slow).
    """
    grid = grid or grid_sizes(k_max, l_max)
    ctx = Assembly(k_max, l_max, gamma, grid, kernel_scale, precision)
    trip = channels(l_max)
    look = {t: i for i, t in enumerate(trip)}
    n_k, n_t = k_max + 1, len(trip)
    need = set(range(n_t)) if only is None else set()
    if only is not None:  # a channel needs its swap partner, whose full needs its own partner
        for i in only:
            l1, l2, l3 = trip[i]
            need |= {i, look[(l1, l3, l2)]}
    gains = np.full((n_t, n_k, n_k, n_k), np.nan)
    losses = np.full_like(gains, np.nan)
    for i in sorted(need):
        g, lf, ls = ctx.channel_half(*trip[i])
        gains[i], losses[i] = g, lf + ls
    full = np.full_like(gains, np.nan)
    for i in need:
        l1, l2, l3 = trip[i]
        s = look[(l1, l3, l2)]
        full[i] = gains[i] + gains[s].transpose(0, 2, 1) - losses[i]
    vals = np.full((n_k, n_k, n_k, n_t), np.nan)
    for i in (need if only is None else only):
        l1, l2, l3 = trip[i]
        s = look[(l1, l3, l2)]
        vals[:, :, :, i] = channel_scale(l1, l2, l3) * (0.5 * (full[i] + full[s].transpose(0, 2, 1)))
    if conservation:
        for i, (l1, _, _) in enumerate(trip):
            if l1 <= 1:
                vals[0, :, :, i] = 0.0
            if l1 == 0 and n_k > 1:
                vals[1, :, :, i] = 0.0
    if detailed_balance:
        vals[:, 0, 0, look[(0, 0, 0)]] = 0.0
    return vals
