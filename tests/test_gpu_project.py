"""GPU projection of drifting Maxwellians (bfq_project_maxwellians) against the
reference's basis.project goldens and the host generator."""

import os

import numpy as np
import pytest
import torch

from conftest import GOLDEN
from paper_2605_28475_b200 import inputs

pytestmark = pytest.mark.gpu


def test_device_projection_matches_reference_project():
    d = np.load(os.path.join(GOLDEN, "project.npz"))
    for i, (k_max, l_max, ux, uy, uz, t) in enumerate(d["meta"]):
        u = torch.tensor([[ux, uy, uz]], dtype=torch.float64, device="cuda")
        tt = torch.tensor([t], dtype=torch.float64, device="cuda")
        mine = inputs.project_maxwellians_device(int(k_max) + 1, int(l_max), u, tt)[0].cpu().numpy()
        assert np.abs(mine - d[f"c{i}"]).max() < 5e-13


@pytest.mark.parametrize("n_k,l_max", [(5, 4), (9, 8), (13, 12), (17, 16)])
def test_device_generator_matches_host_generator(n_k, l_max):
    host = inputs.perturbed_maxwellians(n_k, l_max, 1500, seed=11, start=700)
    dev = inputs.perturbed_maxwellians_device(n_k, l_max, 1500, seed=11, start=700).cpu().numpy()
    assert np.abs(dev - host).max() / np.abs(host).max() < 1e-13
    for k, q in inputs.INVARIANT_SLOTS[1:]:
        # noise-free invariant slots carry the projected moments of the Maxwellian only
        assert np.abs(dev[:, k, q] - host[:, k, q]).max() < 1e-13


def test_device_bimodal_matches_host():
    host = inputs.bimodal(11, 10, 600, seed=5)
    dev = inputs.bimodal_device(11, 10, 600, seed=5).cpu().numpy()
    assert np.abs(dev - host).max() / np.abs(host).max() < 1e-13


def test_zero_drift_and_rejects_bad_shapes():
    u = torch.zeros((3, 3), dtype=torch.float64, device="cuda")
    t = torch.ones(3, dtype=torch.float64, device="cuda")
    c = inputs.project_maxwellians_device(5, 4, u, t).cpu().numpy()
    assert abs(c[0, 0, 0] - 1.0) < 1e-14  # the unit Maxwellian is psi_000
    assert np.abs(c[:, 0, 1:]).max() < 1e-15
    with pytest.raises(ValueError):
        inputs.project_maxwellians_device(5, 4, u[:, :2].contiguous(), t)
