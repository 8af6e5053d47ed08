"""The paper's two-level model Hamiltonian and SP2 on it.

CPU pins: the printed parameter sets, exact symmetry, the metal entry the SPEC derives from the paper
(-1.0 * exp(-0.01 |j - i|) between A orbitals), monotone decay at r = 0, and SP2-Basic (oracle) on the
gapped soft-matter system reaching the eigh projector at tau = 0. GPU: the same SP2 bitwise vs the
oracle at tau = 1e-5 (the gapped system the paper ran ExaSP2 on)."""
import math

import numpy as np
import pytest

import oracle
import synth


def test_presets_are_the_papers():
    P = synth.MODEL_PRESETS
    assert P["metal"] == dict(d_aa=-1.0, d_bb=-1.0, k=-0.01)
    assert P["semiconductor"] == dict(d_bb=-1.0, d_ab_intra=-2.0, k=-0.01)
    assert P["soft_matter"] == dict(d_bb=-1.0, d_ab_intra=-1.0, eps_a=-10.0, k=-0.1, r=1.0)


@pytest.mark.parametrize("kind", ["metal", "semiconductor", "soft_matter"])
def test_exact_symmetry_and_seed_determinism(kind):
    H = synth.model_hamiltonian(512, kind)
    D = H.to_dense()
    assert np.array_equal(D, D.T)
    assert np.array_equal(D, synth.model_hamiltonian(512, kind).to_dense())


def test_metal_entry_between_a_orbitals():
    # SPEC S:L252 example: r = 0 -> H[A_i, A_j] = -1.0 * exp(-0.01 |j - i|), dimer distance
    D = synth.model_hamiltonian(128, "metal", r=0.0).to_dense()
    for d1, d2 in [(0, 1), (3, 17), (10, 63)]:
        assert D[2 * d1, 2 * d2] == -1.0 * math.exp(-0.01 * abs(d2 - d1))  # libm exp, as the generator
        assert D[2 * d1 + 1, 2 * d2 + 1] == -1.0 * math.exp(-0.01 * abs(d2 - d1))
        assert D[2 * d1, 2 * d2 + 1] == 0.0  # no A-B coupling across dimers in the metal preset


def test_decay_is_monotone_without_noise():
    D = synth.model_hamiltonian(256, "soft_matter", r=0.0, tau_store=0.0).to_dense()
    row = np.abs(D[1, 3::2])  # B_0 to B_d, d = 1, 2, ...
    assert np.all(np.diff(row) <= 0) and row[0] == math.exp(-0.1)


def test_soft_matter_sp2_reaches_the_projector():
    n = 512
    H = synth.model_hamiltonian(n, "soft_matter", tau_store=0.0)
    r = oracle.sp2(H, n // 2, 1e-10, oracle.SP2Opts(threshold=0.0, max_iter=100), d_width=n)
    assert r.stop == "CONVERGED"
    D = r.D.to_dense()
    w, v = np.linalg.eigh(H.to_dense())
    P = v[:, : n // 2] @ v[:, : n // 2].T
    assert np.abs(D - P).max() < 1e-8
    assert abs(np.trace(D) - n // 2) < 1e-8


@pytest.mark.gpu
def test_soft_matter_sp2_gpu_bitwise():
    from tests.helpers import same_bits
    from tests.test_gpu_parity import eb, up
    ctx = eb().Context(0)
    n, tau = 2048, 1e-5
    H = synth.model_hamiltonian(n, "soft_matter", tau_store=tau)
    o = oracle.sp2(H, n // 2, 1e-8, oracle.SP2Opts(threshold=tau, max_iter=60), d_width=n)
    assert o.status in (oracle.OK, oracle.NOCONV)
    d = eb().Mat.empty(n, n)
    g = ctx.sp2_run(up(H), n // 2, 1e-8, d, threshold=tau, max_iter=60)
    assert (g.iterations, g.stop, g.trD) == (o.iterations, o.stop, o.trD)
    for a, b in zip(g.iters, o.iters):
        assert (a["branch"], a["trX"], a["trS"], a["e"], a["products"]) == (b["branch"], b["trX"], b["trS"], b["e"],
                                                                            b["products"])
    assert same_bits(d.to_host(), o.D)
    ctx.close()
