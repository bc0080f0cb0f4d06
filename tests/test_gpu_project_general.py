"""General batched projection on the GPU (bfq_project_samples, csrc/
bfq_project_samples.cu) against the live reference's basis.project(f, cfg,
order) outputs (tests/golden/project_general.npz, make_project_golden.py) and
against the closed-form projection of drifting Maxwellians; the single-cell
drop-in project(f, cfg, order); determinism and argument validation."""

import os
import sys

import numpy as np
import pytest

from conftest import GOLDEN

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

sys.path.insert(0, GOLDEN)
from project_funcs import CASES, FUNCS  # noqa: E402

from paper_2605_28475_b200 import inputs  # noqa: E402
from paper_2605_28475_b200 import project as gproject  # noqa: E402
from paper_2605_28475_b200.operator import CoefficientField, SpectralConfig  # noqa: E402

GOLD = np.load(os.path.join(GOLDEN, "project_general.npz"))


def rel(a, b):
    return float(np.max(np.abs(a - b)) / np.max(np.abs(b)))


@pytest.mark.parametrize("case", CASES)
def test_batch_matches_reference_project(case):
    k, l, order = case
    cfg = SpectralConfig(k, l, 1.0)
    pts = gproject.project_points(cfg, order)
    names = sorted(FUNCS)
    samples = np.stack([FUNCS[n](pts) for n in names] * 3)  # 3 copies: ragged-free batch of 9
    pj = gproject.Projector(cfg, order)
    got = pj.project(torch.from_numpy(samples).cuda()).cpu().numpy()
    for i, n in enumerate(names * 3):
        assert rel(got[i], GOLD[f"{n}_k{k}_l{l}_o{order}"]) <= 1e-13, (n, i)
    # bitwise deterministic and position independent
    again = pj.project(torch.from_numpy(samples[::-1].copy()).cuda()).cpu().numpy()[::-1]
    assert np.array_equal(got, again)


def test_maxwellians_match_closed_form():
    cfg = SpectralConfig(12, 12, 1.0)
    order = 64
    pts = torch.from_numpy(gproject.project_points(cfg, order)).cuda()
    rng = np.random.default_rng(3)
    n = 37
    u = rng.uniform(-0.3, 0.3, size=(n, 3))
    t = rng.uniform(0.8, 1.2, size=n)
    ut, tt = torch.from_numpy(u).cuda(), torch.from_numpy(t).cuda()
    d2 = ((pts[None, :, :] - ut[:, None, :]) ** 2).sum(-1)
    samples = (2 * np.pi * tt[:, None]) ** -1.5 * torch.exp(-d2 / (2 * tt[:, None]))
    got = gproject.Projector(cfg, order).project(samples.contiguous()).cpu().numpy()
    ref = inputs.project_maxwellians(cfg.n_k, cfg.l_max, u, t)
    for i in range(n):
        assert rel(got[i], ref[i]) <= 1e-12, i


def test_single_cell_dropin():
    cfg = SpectralConfig(8, 8, 1.0)
    c = gproject.project(FUNCS["quartic"], cfg, 32)
    assert isinstance(c, CoefficientField)
    assert rel(c.values, GOLD["quartic_k8_l8_o32"]) <= 1e-13


def test_validation():
    cfg = SpectralConfig(4, 4, 1.0)
    pj = gproject.Projector(cfg, 16)
    with pytest.raises(ValueError):
        pj.project(torch.zeros((2, pj.n_points + 1), dtype=torch.float64, device="cuda"))
    with pytest.raises(ValueError):
        pj.project(torch.zeros((2, pj.n_points), dtype=torch.float32, device="cuda"))
    with pytest.raises(ValueError):
        pj.project(torch.zeros((2, pj.n_points), dtype=torch.float64))
    assert pj.project(torch.zeros((0, pj.n_points), dtype=torch.float64, device="cuda")).shape == (0, 5, 25)


@pytest.mark.parametrize("case", CASES)
def test_v1_kernel_matches_reference_project(case, monkeypatch):
    """The first-generation kernel (forced with BFQ_PROJ_V1; used for shapes the
    v2 register tiles do not cover) stays on the reference's outputs, and the
    two kernels agree to rounding."""
    k, l, order = case
    cfg = SpectralConfig(k, l, 1.0)
    pts = gproject.project_points(cfg, order)
    names = sorted(FUNCS)
    samples = torch.from_numpy(np.stack([FUNCS[n](pts) for n in names])).cuda()
    v2 = gproject.Projector(cfg, order).project(samples).cpu().numpy()
    monkeypatch.setenv("BFQ_PROJ_V1", "1")
    v1 = gproject.Projector(cfg, order).project(samples).cpu().numpy()
    for i, n in enumerate(names):
        assert rel(v1[i], GOLD[f"{n}_k{k}_l{l}_o{order}"]) <= 1e-13, n
        assert rel(v2[i], v1[i]) <= 1e-14, n


@pytest.mark.parametrize("order,offset", [(13, 1), (13, 0), (80, 1)])
def test_odd_grids_and_misaligned_samples(order, offset):
    """n_t n_p odd (order 13 at L=4: 13 x 27 points per slab) makes the slabs
    alternate between 16-byte aligned and not, with an odd element count and a
    partial polar chunk; a one-double offset of the whole batch shifts every
    slab; order 80 (n_p = 161) exceeds the v2 register tiles (v1 path).  All
    against the CPU restatement of basis.project."""
    from oracle.project_oracle import ProjectionOracle

    cfg = SpectralConfig(4, 4, 1.0)
    pts = gproject.project_points(cfg, order)
    names = sorted(FUNCS)
    host = np.stack([FUNCS[n](pts) for n in names])
    buf = torch.empty(host.size + 1, dtype=torch.float64, device="cuda")
    samples = buf[offset:offset + host.size].view(host.shape)
    samples.copy_(torch.from_numpy(host))
    got = gproject.Projector(cfg, order).project(samples).cpu().numpy()
    orc = ProjectionOracle(cfg.k_max, cfg.l_max, gproject.projection_grid(cfg.l_max, order))
    for i, n in enumerate(names):
        assert rel(got[i], orc.project(host[i])) <= 1e-13, (n, order, offset)


@pytest.mark.parametrize("case", [c for c in CASES if c[1] >= 8])
def test_folded_kernel_matches_reference_and_unfolded(case, monkeypatch):
    """The mirror-folded kernel (kernel 3: K over the sample pairs p, n_p - p) is
    the default at these shapes; it stays on the reference's outputs and agrees
    with the unfolded kernel (BFQ_PROJ_NOFOLD) to rounding."""
    k, l, order = case
    cfg = SpectralConfig(k, l, 1.0)
    pts = gproject.project_points(cfg, order)
    names = sorted(FUNCS)
    samples = torch.from_numpy(np.stack([FUNCS[n](pts) for n in names])).cuda()
    pf = gproject.Projector(cfg, order)
    assert pf.kernel == 3
    fold = pf.project(samples).cpu().numpy()
    # the two-K-part layout of the folded kernel (the default above keeps K whole at these orders)
    monkeypatch.setenv("BFQ_PROJ_FOLD_SPLITK", "1")
    ps = gproject.Projector(cfg, order)
    assert ps.kernel == 3
    split = ps.project(samples).cpu().numpy()
    monkeypatch.setenv("BFQ_PROJ_NOFOLD", "1")
    pu = gproject.Projector(cfg, order)
    assert pu.kernel == 2
    plain = pu.project(samples).cpu().numpy()
    for i, n in enumerate(names):
        assert rel(fold[i], GOLD[f"{n}_k{k}_l{l}_o{order}"]) <= 1e-13, n
        assert rel(split[i], GOLD[f"{n}_k{k}_l{l}_o{order}"]) <= 1e-13, n
        assert rel(fold[i], plain[i]) <= 5e-14, n
        assert rel(fold[i], split[i]) <= 1e-14, n


@pytest.mark.parametrize("l_max,order,offset", [(8, 48, 0), (8, 48, 1), (14, 32, 1), (9, 64, 0), (8, 80, 1), (8, 16, 0)])
def test_folded_kernel_partial_chunks_and_misaligned(l_max, order, offset):
    """Folded kernel on a partial polar chunk with unequal K parts (order 48: 48 =
    32 + 16 polar rows, three 16-pair blocks split 1 + 2), on the widest |m| tile
    pair the epilogue holds (l_max = 14) and on a half-empty one (l_max = 9), with the batch shifted
    by one double; order 80 (five 16-pair blocks) takes the two-K-part layout,
    order 16 a single block; against the CPU restatement of basis.project."""
    from oracle.project_oracle import ProjectionOracle

    cfg = SpectralConfig(3, l_max, 1.0)
    pts = gproject.project_points(cfg, order)
    names = sorted(FUNCS)
    # plus white noise: every (v, t) slab and every sample pair carries weight (the
    # test functions decay at large v and would hide an error there)
    host = np.stack([FUNCS[n](pts) for n in names] + [np.random.default_rng(5).standard_normal(pts.shape[0])])
    buf = torch.empty(host.size + 1, dtype=torch.float64, device="cuda")
    samples = buf[offset:offset + host.size].view(host.shape)
    samples.copy_(torch.from_numpy(host))
    pj = gproject.Projector(cfg, order)
    assert pj.kernel == 3
    got = pj.project(samples).cpu().numpy()
    orc = ProjectionOracle(cfg.k_max, cfg.l_max, gproject.projection_grid(cfg.l_max, order))
    for i in range(host.shape[0]):
        assert rel(got[i], orc.project(host[i])) <= 1e-13, (i, l_max, order, offset)


def test_asymmetric_azimuth_table_keeps_the_unfolded_kernel():
    """bfq_projector_create folds only a table that is even / odd under the mirror:
    a perturbed table (C ABI) falls back to kernel 2."""
    import ctypes

    from paper_2605_28475_b200 import _lib

    cfg = SpectralConfig(8, 8, 1.0)
    phi_tab, theta_tab, radial_tab, (n_v, n_t, n_p) = gproject.projection_tables(cfg, 32)
    lib = _lib.lib()
    f64p = ctypes.POINTER(ctypes.c_double)
    kinds = []
    for bump in (0.0, 1e-9):
        tab = phi_tab.copy()
        tab[4, 3] += bump
        h = ctypes.c_void_p()
        _lib.check(lib.bfq_projector_create(cfg.k_max, cfg.l_max, n_v, n_t, n_p, tab.ctypes.data_as(f64p),
                                            theta_tab.ctypes.data_as(f64p), radial_tab.ctypes.data_as(f64p),
                                            torch.cuda.current_device(), ctypes.byref(h)))
        kinds.append(int(lib.bfq_projector_kernel(h)))
        lib.bfq_projector_destroy(h)
    assert kinds == [3, 2]


@pytest.mark.parametrize("l_max,order", [(8, 32), (8, 48), (4, 16)])
def test_persistent_ctas_are_position_independent(l_max, order):
    """The v2 kernels run one CTA per SM over cells blockIdx.x, + gridDim.x, ... with the
    sample ring and the barrier phases carried across cell boundaries: a batch of more
    than two cells per SM (ragged) must give every cell bitwise the result it gets in a
    batch of its own (one cell per CTA)."""
    cfg = SpectralConfig(3, l_max, 1.0)
    pts = gproject.project_points(cfg, order)
    names = sorted(FUNCS)
    rng = np.random.default_rng(11)
    base = np.stack([FUNCS[n](pts) for n in names] + [rng.standard_normal(pts.shape[0])])
    pj = gproject.Projector(cfg, order)
    alone = pj.project(torch.from_numpy(base).cuda())
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    n = 2 * sms + 5
    idx = rng.integers(0, base.shape[0], size=n)
    big = torch.from_numpy(base).cuda()[torch.from_numpy(idx).cuda()].contiguous()
    got = pj.project(big)
    assert torch.equal(got, alone[torch.from_numpy(idx).cuda()])
