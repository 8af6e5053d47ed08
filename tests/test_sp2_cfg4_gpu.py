"""cfg4 (BASELINE configs[3]: 32^3 lattice x 2 orbitals, N = 65536, M = 256, tau = 1e-5) on the GPU:
the literal width-256 run overflows where the oracle does (SURVEY §8d "SP2 protocol", cfg4
literal run), and a 2-iteration GROW window matches the oracle iterate by iterate."""
import numpy as np
import pytest

import oracle
import synth
from tests.helpers import same_bits
from tests.test_gpu_parity import eb, up


@pytest.mark.gpu
def test_sp2_cfg4_literal_overflow_and_window(ctx):
    H = synth.cfg4()
    cf = synth.CFG4
    of = oracle.sp2(H, cf["nocc"], cf["tol"], oracle.SP2Opts(threshold=cf["threshold"], on_overflow=0),
                    d_width=256)
    d = eb().Mat.empty(H.n, 256)
    gf = ctx.sp2_run(up(H), cf["nocc"], cf["tol"], d, threshold=cf["threshold"], on_overflow=eb().SP2_FAIL)
    assert of.status == oracle.OVERFLOW and gf.status == eb().ERR_OVERFLOW
    assert (gf.fail_iter, gf.required_width, gf.overflow_rows) == (of.fail_iter, of.required_width,
                                                                  of.overflow_rows)
    og = oracle.sp2(H, cf["nocc"], cf["tol"], oracle.SP2Opts(threshold=cf["threshold"], max_iter=2), d_width=1024)
    d = eb().Mat.empty(H.n, 1024)
    gg = ctx.sp2_run(up(H), cf["nocc"], cf["tol"], d, threshold=cf["threshold"], max_iter=2)
    assert gg.iterations == og.iterations == 2 and gg.stop == og.stop
    assert gg.regrows == og.regrows and gg.final_width == og.final_width
    for a, b in zip(gg.iters, og.iters):
        assert (a["branch"], a["trX"], a["trS"], a["e"]) == (b["branch"], b["trX"], b["trS"], b["e"])
        assert (a["width"], a["required"], a["products"]) == (b["width"], b["required"], b["products"])
    assert same_bits(d.to_host(), og.D)
