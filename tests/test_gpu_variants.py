"""Round-2 production variants against the paths they replaced (environment
switches read at context creation): bitwise where the
arithmetic is identical, to round-off where it is not.

* IBMG_DF_ES: the dataflow sweep with one E'-row slot and the inverse in
  registers (2 CTAs/SM) runs big_block_es with the same summation order as
  the slab-slot big_block_slab: bitwise.
* IBMG_SPEC: the speculative next V-cycle behind the FGMRES dots computes the
  same column as the non-speculative one: bitwise steps.
* IBMG_CANON_INV: canonical-order inverses are the same inverses, permuted:
  bitwise.
* IBMG_GF: gather-first fused apply / restriction add the same sign * L F to
  the same grid value (v + s either way): bitwise.
* IBMG_GJ256: the register-resident in-place Gauss-Jordan and the 256-thread
  [A | I] form invert the same boxes with different operation orders:
  round-off (the V-cycle to 1e-12, the step to 1e-10, same iterations).
"""
import os

import numpy as np
import pytest

from helpers import rand, rel
from paper_1311_5614_b200 import configs
from paper_1311_5614_b200.ibmg import SaddleSystem

pytestmark = pytest.mark.gpu


def make(prob, **env):
    old = {k: os.environ.get(k) for k in env}
    os.environ.update({k: str(v) for k, v in env.items()})
    try:
        return SaddleSystem.from_problem(prob)
    finally:
        for k, v in old.items():
            if v is None:
                del os.environ[k]
            else:
                os.environ[k] = v


def step(g, prob):
    n = prob.N
    u, p, X = np.zeros(2 * n * n), np.zeros(n * n), prob.X.reshape(-1).copy()
    st = g.step_implicit(u, p, X)
    return u, p, X, st


@pytest.mark.parametrize("var,a,b,bitwise", [
    ("IBMG_DF_ES", 1, 0, True),
    ("IBMG_SPEC", 1, 0, True),
    ("IBMG_CANON_INV", 1, 0, True),
    ("IBMG_GJ256", 0, 1, False),
    ("IBMG_GF", 1, 0, True),  # (opt-in)
])
def test_variant_step(var, a, b, bitwise):
    prob = configs.config2(1e6)
    ga, gb = make(prob, **{var: a}), make(prob, **{var: b})
    ua, pa, Xa, sa = step(ga, prob)
    ub, pb, Xb, sb = step(gb, prob)
    assert sa["converged"] and sb["converged"]
    assert sa["iters"] == sb["iters"]
    if bitwise:
        assert np.array_equal(ua, ub) and np.array_equal(pa, pb) and np.array_equal(Xa, Xb)
    else:
        assert rel(ua, ub) < 1e-10 and rel(pa, pb) < 1e-10 and rel(Xa, Xb) < 1e-14
    ga.close()
    gb.close()


def test_tma_staging_c3_bitwise():
    """IBMG_TMA: the band-major plain phase (levels n > 512; C3's level 1024)
    staging interior tiles' w regions with tensor copies moves the same bytes
    into the same layout: the V-cycle and the step are bitwise equal."""
    prob = configs.config3()
    ga, gb = make(prob, IBMG_TMA=1), make(prob, IBMG_TMA=0)
    b = ga.build_rhs(rand(2 * prob.N ** 2, seed=4))
    assert np.array_equal(ga.v_cycle(b), gb.v_cycle(b))
    ua, pa, Xa, sa = step(ga, prob)
    ub, pb, Xb, sb = step(gb, prob)
    assert sa["iters"] == sb["iters"] and np.array_equal(ua, ub) and np.array_equal(Xa, Xb)
    ga.close()
    gb.close()


def test_register_gauss_jordan_vcycle_c3():
    """C3 (dense coarse levels, 4.8k boxes): the V-cycle with the register
    inverses equals the [A | I] inverses' to round-off."""
    prob = configs.config3()
    ga, gb = make(prob, IBMG_GJ256=0), make(prob, IBMG_GJ256=1)
    b = ga.build_rhs(rand(2 * prob.N ** 2, seed=9))
    assert rel(ga.v_cycle(b), gb.v_cycle(b)) < 1e-12
    ga.close()
    gb.close()


def test_warp_specialised_plain_phase_c3_bitwise():
    """IBMG_PDF2 (default 1): the band-major plain phase with a loader warp feeding three compute
    warps per CTA (k_plain_df2) runs the same tasks in the same order with the same arithmetic as
    the one-warp-per-tile kernel (IBMG_PDF2=0): the V-cycle and the step are bitwise equal (C3's
    level 1024)."""
    prob = configs.config3()
    ga, gb = make(prob, IBMG_PDF2=1), make(prob, IBMG_PDF2=0)
    b = ga.build_rhs(rand(2 * prob.N ** 2, seed=5))
    assert np.array_equal(ga.v_cycle(b), gb.v_cycle(b))
    ua, pa, Xa, sa = step(ga, prob)
    ub, pb, Xb, sb = step(gb, prob)
    assert sa["iters"] == sb["iters"] and np.array_equal(ua, ub) and np.array_equal(Xa, Xb)
    ga.close()
    gb.close()
