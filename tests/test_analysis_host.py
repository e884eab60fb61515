"""Analysis module known answers (acceptance criteria 3-5):
ai_spatial, the naive time-tiled estimate, face sizes, boundary fractions,
their union, the three tight-bound cases and the roofline / ridge point."""
import pytest

import paper_1806_08299_b200 as P
from paper_1806_08299_b200 import analysis as A


def spec(ndims, nterms, dt=1, radius=1):
    terms = []
    for k in range(nterms):
        off = [0] * ndims
        off[k % ndims] = radius if k else 0
        terms.append(P.StencilTerm(0.1, dt if k == nterms - 1 else 1, tuple(off)))
    return P.StencilSpec.make("s", ndims, terms)


def test_ai_spatial_and_naive():
    assert A.ai_spatial(spec(2, 5)) == pytest.approx(9 / 8)
    assert A.ai_spatial(spec(1, 1, radius=0)) == pytest.approx(0.125)
    assert A.ai_spatial(spec(3, 13, dt=2)) == pytest.approx(25 / 12)
    assert A.naive_from_spatial(4.69, 2) == pytest.approx(9.38)
    assert A.naive_from_spatial(4.69, 4) == pytest.approx(18.76)
    s = spec(2, 5)
    assert A.ai_naive_tt(s, 1) == A.ai_spatial(s)
    assert A.bytes_per_point(s) == 8.0


def test_face_sizes_and_fracs():
    s = spec(2, 5)
    assert A.face_sizes(s, (16, 16), 1, (4, 4)) == [32, 8]
    assert A.face_sizes(s, (16, 16), 2, (4, 4)) == [64, 16]
    assert A.boundary_fracs(s, (64, 64), (8, 8)) == [0.25, 0.25]
    s8 = P.StencilSpec.make("r8", 1, [P.StencilTerm(1.0, 1, (8,))])
    assert A.boundary_fracs(s8, (16,), (2,)) == [1.0]
    assert A.union_frac([0.25, 0.1]) == pytest.approx(0.325)
    assert A.union_frac([0.3]) == pytest.approx(0.3)
    assert A.union_frac([]) == 0.0


@pytest.mark.parametrize("omega,case,divisor", [(300, "empty", 1.0), (100, "f1_only", 1 + 1248 / 4096),
                                                (30, "multi", 1.25)])
def test_tight_bound_cases(omega, case, divisor):
    s = spec(2, 5)
    est, faces = A.tight_bound(s, (64, 64), 2, (8, 8), omega)
    assert faces.face_sizes == [256, 32]
    assert faces.bcase == case
    assert est.divisor == pytest.approx(divisor, abs=1e-3)
    assert est.ai_tight_tt == pytest.approx(est.ai_naive_tt / divisor)
    assert est.ai_tight_tt <= est.ai_naive_tt


def test_roofline_and_ridge():
    m = A.MachineProfile(262.01, 17.3)
    assert A.roofline_bound(m, 10) == pytest.approx(173.0, abs=0.01)
    assert A.roofline_bound(m, 20) == pytest.approx(262.01)
    assert A.ridge_point(m) == pytest.approx(15.145, abs=0.01)
    r = A.ridge_point(m)
    assert A.roofline_bound(m, r) == pytest.approx(m.peak_gflops)
