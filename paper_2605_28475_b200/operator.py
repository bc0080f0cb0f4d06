"""Host-side mirror of the reference's operator data model.

The GPU box has no copy of the reference package, so the engine carries its
own minimal, attribute-compatible versions of the containers the hot path
consumes.  Attribute names, index conventions and error types follow the
reference so that either object can be handed to :mod:`.engine`:

* ``SpectralConfig``     -- basis.py:42-66
* ``q_index/q_degree``   -- basis.py:69-81 (1-based q = l^2 + l + m + 1)
* ``CoefficientField``   -- basis.py:210-236 (values (n_k, n_q) float64)
* ``moments``            -- basis.py:346-363
* ``ChannelTable``       -- angular.py:100-135
* ``GauntCOO``           -- angular.py:207-249 (1-based int32 columns)
* ``RTensor``            -- kinematic.py:241-255
* ``FactorizedOperator`` -- contraction.py:76-108 (validation, 0-based views)
* ``load_cache``         -- cache.py:92-166 (BFCT reader, CRC-32 checked)
* ``save_cache``         -- cache.py:52-89 (BFCT writer, same layout)
"""

from __future__ import annotations

import math
import struct
import zlib
from dataclasses import dataclass, field

import numpy as np

__all__ = [
    "SpectralConfig",
    "CoefficientField",
    "ChannelTable",
    "GauntCOO",
    "RTensor",
    "FactorizedOperator",
    "CacheFormatError",
    "CacheIntegrityError",
    "q_index",
    "q_degree",
    "moments",
    "load_cache",
    "save_cache",
]


@dataclass(frozen=True)
class SpectralConfig:
    k_max: int
    l_max: int
    gamma: float = 1.0

    def __post_init__(self):
        if self.k_max < 0 or self.l_max < 0:
            raise ValueError("truncation limits must be non-negative")
        if not 0.0 <= self.gamma <= 1.0:
            raise ValueError(f"kernel exponent gamma={self.gamma} outside [0, 1]")

    @property
    def n_k(self) -> int:
        return self.k_max + 1

    @property
    def n_q(self) -> int:
        return (self.l_max + 1) ** 2

    @property
    def n_dof(self) -> int:
        return self.n_k * self.n_q


def q_index(l: int, m: int) -> int:
    if l < 0 or abs(m) > l:
        raise ValueError(f"invalid angular numbers l={l}, m={m}")
    return l * (l + 1) + m + 1


def q_degree(q: int) -> tuple[int, int]:
    if q < 1:
        raise ValueError(f"angular index must be >= 1, got {q}")
    l = math.isqrt(q - 1)
    return l, q - 1 - l * (l + 1)


@dataclass
class CoefficientField:
    values: np.ndarray
    cfg: SpectralConfig = field(repr=False)

    def __post_init__(self):
        shape = (self.cfg.n_k, self.cfg.n_q)
        if self.values.shape != shape:
            raise ValueError(f"coefficient array must have shape {shape}")

    @classmethod
    def zeros(cls, cfg: SpectralConfig) -> "CoefficientField":
        return cls(np.zeros((cfg.n_k, cfg.n_q)), cfg)

    @classmethod
    def equilibrium(cls, cfg: SpectralConfig) -> "CoefficientField":
        out = cls.zeros(cfg)
        out.values[0, 0] = 1.0
        return out

    def copy(self) -> "CoefficientField":
        return CoefficientField(self.values.copy(), self.cfg)


_SQRT6 = math.sqrt(6.0)


def moments(c) -> tuple[float, np.ndarray, float]:
    """Mass, momentum (x, y, z) and kinetic energy of one field.

    Momentum components are the (l=1, m=+1), (1, -1), (1, 0) modes at k=0,
    energy is (3 c_000 - sqrt(6) c_100) / 2 (basis.py:340-363).
    """
    v = c.values
    l_max = c.cfg.l_max
    mass = v[0, 0]
    mom = np.array([v[0, 3], v[0, 1], v[0, 2]]) if l_max >= 1 else np.zeros(3)
    e2 = v[1, 0] if c.cfg.k_max >= 1 else 0.0
    return float(mass), mom, float(0.5 * (3.0 * mass - _SQRT6 * e2))


@dataclass(frozen=True)
class ChannelTable:
    l_max: int
    triplets: tuple
    _lookup: dict = field(repr=False, hash=False, compare=False)

    @property
    def n_t(self) -> int:
        return len(self.triplets)

    def tau(self, l1: int, l2: int, l3: int) -> int:
        return self._lookup[(l1, l2, l3)]

    def triplet(self, tau: int) -> tuple:
        return self.triplets[tau - 1]

    @classmethod
    def from_triplets(cls, l_max: int, triplets) -> "ChannelTable":
        trip = tuple(tuple(int(x) for x in t) for t in triplets)
        return cls(l_max, trip, {t: i + 1 for i, t in enumerate(trip)})


@dataclass
class GauntCOO:
    l_max: int
    n_q: int
    channels: ChannelTable
    q1: np.ndarray
    q2: np.ndarray
    q3: np.ndarray
    tau: np.ndarray
    g: np.ndarray
    slice_starts: np.ndarray
    slice_tau: np.ndarray
    slice_q1: np.ndarray

    @property
    def n_g(self) -> int:
        return self.g.size

    @property
    def n_s(self) -> int:
        return self.slice_tau.size


@dataclass
class RTensor:
    values: np.ndarray  # (n_k, n_k, n_k, N_T) float64, C-order
    channels: ChannelTable
    gamma: float
    grid: tuple = ()
    conservation_applied: bool = False
    detailed_balance_applied: bool = False
    max_zeroed: float = 0.0  # largest magnitude overwritten by the corrections

    @property
    def n_k(self) -> int:
        return self.values.shape[0]


@dataclass
class FactorizedOperator:
    r: RTensor
    g: GauntCOO
    cfg: SpectralConfig

    def __post_init__(self):
        if self.g.l_max != self.cfg.l_max:
            raise ValueError("routing table and configuration disagree on l_max")
        if self.r.values.shape != (self.cfg.n_k,) * 3 + (self.g.channels.n_t,):
            raise ValueError("physical tensor shape inconsistent with table")
        if self.g.tau.min() < 1 or self.g.tau.max() > self.g.channels.n_t:
            raise ValueError("channel index out of range")
        for col in (self.g.q1, self.g.q2, self.g.q3):
            if col.min() < 1 or col.max() > self.cfg.n_q:
                raise ValueError("angular index out of range")
        if self.g.n_s > self.g.n_g:
            raise ValueError("slice count cannot exceed row count")
        self.q1_0 = self.g.q1.astype(np.int64) - 1
        self.q2_0 = self.g.q2.astype(np.int64) - 1
        self.q3_0 = self.g.q3.astype(np.int64) - 1
        self.tau_0 = self.g.tau.astype(np.int64) - 1
        self.slice_tau_0 = self.g.slice_tau.astype(np.int64) - 1
        self.slice_q1_0 = self.g.slice_q1.astype(np.int64) - 1

    @property
    def n_s(self) -> int:
        return self.g.n_s


# ---------------------------------------------------------------- BFCT cache
class CacheFormatError(RuntimeError):
    """Unrecognized or incompatible cache layout (cache.py:32-33)."""


class CacheIntegrityError(RuntimeError):
    """Payload does not match its checksum or advertised sizes (cache.py:36-37)."""


_MAGIC = b"BFCT"
_HDR = struct.Struct("<4sIIId9IIQII")  # cache.py:41


def slices_from_rows(tau: np.ndarray, q1: np.ndarray, n_q: int):
    """(tau, q1) slice starts of a sorted table (cache.py:147-150)."""
    key = tau.astype(np.int64) * n_q + (q1.astype(np.int64) - 1)
    starts = np.concatenate(([0], np.flatnonzero(np.diff(key)) + 1, [key.size])).astype(np.int64)
    return starts, tau[starts[:-1]].copy(), q1[starts[:-1]].copy()


def load_cache(path) -> FactorizedOperator:
    """Read a BFCT operator file written by the reference's ``save_cache``."""
    with open(path, "rb") as fh:
        blob = fh.read()
    if len(blob) < _HDR.size:
        raise CacheFormatError("file too short for a cache header")
    (magic, version, k_max, l_max, gamma, *rest) = _HDR.unpack_from(blob)
    grid = tuple(rest[:9])
    n_t, n_g, flags, crc = rest[9], rest[10], rest[11], rest[12]
    if magic != _MAGIC:
        raise CacheFormatError(f"bad magic {magic!r}")
    if version != 1:
        raise CacheFormatError(f"cache format version {version} unsupported (expected 1)")
    payload = memoryview(blob)[_HDR.size:]
    if zlib.crc32(payload) & 0xFFFFFFFF != crc:
        raise CacheIntegrityError("payload checksum mismatch")
    n_k = k_max + 1
    want = 12 * n_t + 24 * n_g + 8 * n_k**3 * n_t
    if len(payload) != want:
        raise CacheIntegrityError(f"payload size {len(payload)} != expected {want}")
    pos = 0

    def take(dt, count):
        nonlocal pos
        out = np.frombuffer(payload, dtype=dt, count=count, offset=pos)
        pos += out.nbytes
        return out

    triplets = take("<u4", 3 * n_t).reshape(n_t, 3).astype(int)
    cols = [take("<u4", n_g).astype(np.int32) for _ in range(4)]
    q1, q2, q3, tau = cols
    g = take("<f8", n_g).astype(np.float64)
    values = take("<f8", n_k**3 * n_t).astype(np.float64).reshape(n_k, n_k, n_k, n_t)
    channels = ChannelTable.from_triplets(l_max, [tuple(t) for t in triplets])
    n_q = (l_max + 1) ** 2
    starts, s_tau, s_q1 = slices_from_rows(tau, q1, n_q)
    coo = GauntCOO(l_max, n_q, channels, q1, q2, q3, tau, g, starts, s_tau, s_q1)
    r = RTensor(values, channels, gamma, grid, bool(flags & 1), bool(flags & 2))
    return FactorizedOperator(r, coo, SpectralConfig(k_max, l_max, gamma))


def save_cache(path, op: FactorizedOperator) -> int:
    """Serialise an operator in the reference's BFCT layout (cache.py:52-89);
    returns the number of bytes written.  The reference's ``load_cache`` reads it."""
    chans = np.asarray(op.g.channels.triplets, dtype="<u4")
    payload = b"".join([
        chans.tobytes(),
        *(np.asarray(c).astype("<u4").tobytes() for c in (op.g.q1, op.g.q2, op.g.q3, op.g.tau)),
        np.asarray(op.g.g).astype("<f8").tobytes(),
        np.ascontiguousarray(op.r.values).astype("<f8").tobytes(),
    ])
    flags = (1 if op.r.conservation_applied else 0) | (2 if op.r.detailed_balance_applied else 0)
    g = op.r.grid
    grid = tuple(g.as_tuple()) if hasattr(g, "as_tuple") else (tuple(g) if g else (0,) * 9)
    if len(grid) != 9:
        raise ValueError("operator grid spec must have 9 entries")
    header = _HDR.pack(_MAGIC, 1, op.cfg.k_max, op.cfg.l_max, float(op.cfg.gamma), *grid,
                       op.g.channels.n_t, op.g.n_g, flags, zlib.crc32(payload) & 0xFFFFFFFF)
    with open(path, "wb") as fh:
        fh.write(header)
        fh.write(payload)
    return len(header) + len(payload)
