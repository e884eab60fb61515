"""CPU tests of the drop-in boundary: the C-ABI library loads and exports
every symbol include/stencil_tiler.h declares, its host-side logic (spec
model, parse_spec, legality, slots, initialisers, verify_bitwise) matches the
reference contract and the oracle, and the C++ mirror (tiler_gpu.hpp)
compiles and runs its host checks.  No GPU compute here."""
import ctypes as C
import os
import re
import subprocess

import numpy as np
import pytest

import _oracle as O
import paper_1806_08299_b200 as P
from paper_1806_08299_b200 import _native as N
from paper_1806_08299_b200 import configs as CF

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "stencil_tiler.h")


def declared_symbols():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(st_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    lib = C.CDLL(N.LIB_PATH)
    syms = declared_symbols()
    assert len(syms) >= 35
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing
    # and the ctypes table covers them all
    assert sorted(n for n, _, _ in N.SIGNATURES) == syms


def test_version_and_error_string():
    lib = N.load()
    assert b"sm_100a" in lib.st_version()
    h = C.c_void_p()
    rc = lib.st_stencil_create(b"x", 4, None, 0, 0, C.byref(h))
    assert rc == P.tiler.ST_ERR_INVALID and b"ndims" in lib.st_last_error()


def test_spec_model_known_answers():
    # SPEC.md:54-83 examples
    s, sp = P.parse_spec("stencil s\ndims 1\nextent 8\nsteps 4\nterm 1.0 1 0")
    assert s.ndims == 1 and s.time_depth == 1 and s.radii == [0] and sp == P.IterationSpace(4, (8,))
    s2, _ = P.parse_spec("stencil s\ndims 1\nextent 8\nsteps 4\nterm 0.5 1 -1\nterm 0.5 1 1")
    assert s2.radii == [1] and s2.time_depth == 1
    with pytest.raises(P.ParseError) as e:
        P.parse_spec("stencil s\ndims 1\nextent 8\nsteps 4\nterm 1.0 0 0")
    assert e.value.line() == 5
    s3 = P.StencilSpec.make("s", 3, [P.StencilTerm(0.1, 1, (2, 0, 0)), P.StencilTerm(0.1, 1, (0, 1, 0)),
                                     P.StencilTerm(0.1, 1, (0, 0, 2))])
    assert P.min_skew_factor(s3) == 2
    assert P.min_skew_factor(P.StencilSpec.make("z", 1, [P.StencilTerm(1.0, 1, (0,))])) == 0
    assert P.time_buffer_slots(s2, 1) == 2 and P.time_buffer_slots(s2, 4) == 5
    s_dt2 = P.StencilSpec.make("d", 1, [P.StencilTerm(0.5, 2, (0,))])
    assert P.time_buffer_slots(s_dt2, 16) == 18
    for k, f in [(1, 1), (3, 5), (7, 13)]:
        sk = P.StencilSpec.make("k", 1, [P.StencilTerm(0.1, 1, (0,))] * k)
        assert P.flops_per_point(sk) == f


@pytest.mark.parametrize("text,line", [
    ("dims 1\nextent 8\nsteps 4\nterm 1 1 0", 5),                     # missing stencil line (end)
    ("stencil s\ndims 4\n", 2),                                        # bad dims
    ("stencil s\ndims 2\nextent 8\n", 3),                              # arity
    ("stencil s\ndims 1\nextent 0\n", 3),                              # non-positive extent
    ("stencil s\ndims 1\nextent 8\nsteps 2\nterm 1 1 0 0\n", 5),       # offsets arity
    ("stencil s\ndims 1\nextent 8\nsteps 2\nbogus 1\n", 5),            # unknown keyword
    ("stencil s\ndims 1\nextent 8\nsteps 2\n", 5),                     # no terms
])
def test_parse_errors_carry_line(text, line):
    with pytest.raises(P.ParseError) as e:
        P.parse_spec(text)
    assert e.value.line() == line


def test_legality_and_required_slots():
    s = P.StencilSpec.make("s", 2, [P.StencilTerm(0.5, 1, (2, 0)), P.StencilTerm(0.5, 1, (0, 2))])
    assert P.check_legality(s, P.TilePlan(2, 2, (4, 4))) is None
    v = P.check_legality(s, P.TilePlan(1, 2, (4, 4)))
    assert v == P.LegalityViolation(1, 2)
    with pytest.raises(P.Error) as e:
        P.tile_time(P.build_canonical_nest(s, None), s, None, P.TilePlan(1, 2, (4, 4)))
    assert e.value.code == P.tiler.ST_ERR_ILLEGAL_PLAN
    canon = P.build_canonical_nest(s, None)
    assert P.required_slots(canon, s) == 2
    assert P.required_slots(P.tile_space_minmax(canon, (4, 4)), s) == 2
    assert P.required_slots(P.tile_time(canon, s, None, P.TilePlan(2, 8, (4, 4))), s) == 9


def _spec_pair(ndims, terms, model=0):
    return O.Spec(ndims, terms, model), P.StencilSpec.make("t", ndims, [P.StencilTerm(c, dt, o) for c, dt, o in terms],
                                                           model=model)


@pytest.mark.parametrize("ndims,ext", [(1, (37,)), (2, (9, 13)), (3, (5, 7, 11))])
def test_product_initialisers_match_oracle(ndims, ext):
    terms = [(0.5, 2, tuple(0 for _ in range(ndims)))] + [
        (0.25, 1, tuple(2 if i == d else 0 for i in range(ndims))) for d in range(ndims)]
    o, p = _spec_pair(ndims, terms)
    slots = 4
    lib = N.load()
    for seed in (0, 7, 123456789):
        a = O.init_reference(o, ext, slots, seed)
        b = np.zeros_like(a)
        assert lib.st_init_reference(p.handle, N.i64array(ext), P.tiler._fptr(b), slots, seed) == 0
        assert np.array_equal(a.view(np.uint32), b.view(np.uint32))
        a = O.init_unit(o, ext, slots, seed)
        b = np.zeros_like(a)
        assert lib.st_init_unit(p.handle, N.i64array(ext), P.tiler._fptr(b), slots, seed) == 0
        assert np.array_equal(a.view(np.uint32), b.view(np.uint32))
    c = [e // 2 for e in ext]
    a = O.init_gaussian(o, ext, slots, 2.5, c)
    b = np.zeros_like(a)
    assert lib.st_init_gaussian(p.handle, N.i64array(ext), P.tiler._fptr(b), slots, 2.5, N.i64array(c)) == 0
    assert np.array_equal(a.view(np.uint32), b.view(np.uint32))


def test_product_fields_match_oracle():
    lib = N.load()
    ext = (6, 9, 11)
    a = O.mfield_layered(ext, 1500.0, 3000.0, 3, 1e-3, 10.0)
    b = np.zeros_like(a)
    assert lib.st_field_layered(3, N.i64array(ext), P.tiler._fptr(b), 1500.0, 3000.0, 3, 1e-3, 10.0, 0) == 0
    assert np.array_equal(a, b)
    a = O.mfield_random(ext, 8299, 1500.0, 4500.0, 8e-4, 10.0)
    b = np.zeros_like(a)
    assert lib.st_field_random_smoothed(3, N.i64array(ext), P.tiler._fptr(b), 8299, 1500.0, 4500.0, 8e-4, 10.0) == 0
    assert np.array_equal(a.view(np.uint32), b.view(np.uint32))


def test_large_parallel_lcg_jump_ahead_matches_sequential():
    # st_init_* fill in parallel with LCG jump-ahead; must equal the stream
    o, p = _spec_pair(3, [(1.0, 1, (0, 0, 0))])
    ext = (40, 50, 60)
    a = O.init_unit(o, ext, 2, 99)
    b = np.zeros_like(a)
    assert N.load().st_init_unit(p.handle, N.i64array(ext), P.tiler._fptr(b), 2, 99) == 0
    assert np.array_equal(a.view(np.uint32), b.view(np.uint32))


def test_verify_bitwise_host():
    o, p = _spec_pair(2, [(0.5, 1, (0, 0)), (0.5, 1, (1, 0))])
    ext = (4, 6)
    a = O.init_reference(o, ext, 2, 1)
    b = a.copy()
    eq = C.c_int()
    lib = N.load()
    assert lib.st_verify_bitwise(p.handle, N.i64array(ext), P.tiler._fptr(a), 2, P.tiler._fptr(b), 2, 1, 2,
                                 C.byref(eq)) == 0 and eq.value == 1
    pv = b.reshape(2, 6, 6)
    pv[1, 2, 2] = np.nextafter(pv[1, 2, 2], np.float32(1))
    assert lib.st_verify_bitwise(p.handle, N.i64array(ext), P.tiler._fptr(a), 2, P.tiler._fptr(b), 2, 1, 2,
                                 C.byref(eq)) == 0 and eq.value == 0
    # not retained -> error (executor.hpp:107-110)
    assert lib.st_verify_bitwise(p.handle, N.i64array(ext), P.tiler._fptr(a), 2, P.tiler._fptr(b), 2, 1, 3,
                                 C.byref(eq)) == P.tiler.ST_ERR_SLOTS


def test_context_without_gpu_fails_cleanly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    h = C.c_void_p()
    rc = N.load().st_context_create(0, C.byref(h))
    assert rc in (P.tiler.ST_ERR_CUDA, P.tiler.ST_ERR_INVALID)
    assert N.load().st_last_error()


def test_config_coefficients_folded_in_double():
    # ledger A.2: 1 - 4*0.2 folded in double, cast once
    c1 = CF.get(1)
    assert np.float32(c1.terms[0][0]) == np.float32(1.0 - 4 * 0.2)
    assert np.float32(c1.terms[0][0]).view(np.uint32) != np.float32(np.float32(1) - np.float32(4) * np.float32(0.2)).view(np.uint32)
    c3 = CF.get(3)
    w = CF.fd2_weights(8)
    assert [float(x) for x in w] == pytest.approx([-205 / 72, 8 / 5, -1 / 5, 8 / 315, -1 / 560])
    assert len(c3.terms) == 25 and len(CF.get(4).terms) == 49
    # canonical star order: centre, then d_1 (-1,+1,-2,+2..), d_2, d_3
    assert [t[2] for t in c3.terms[:5]] == [(0, 0, 0), (-1, 0, 0), (1, 0, 0), (-2, 0, 0), (2, 0, 0)]
    # stability: Courant numbers below the leapfrog limits
    assert max(c3.v_top, c3.v_bottom) * c3.dt / CF.H == pytest.approx(0.4)


def test_cpp_mirror_compiles_and_runs_host_checks(tmp_path):
    exe = tmp_path / "test_tiler_api"
    libdir = os.path.dirname(N.LIB_PATH)
    subprocess.run(["/usr/bin/g++", "-std=c++17", "-O1", "-I" + os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "cpp", "test_tiler_api.cpp"), "-L" + libdir, "-lstencil_tiler",
                    "-Wl,-rpath," + libdir, "-o", str(exe)], check=True)
    out = subprocess.run([str(exe)], check=True, capture_output=True, text=True).stdout
    assert "host checks ok" in out


def test_study_workloads_defined_like_the_configs():
    """Study workloads 6 and 7 (beyond BASELINE's five): the same operator
    families, coefficients folded in double and cast once, stable."""
    c6 = CF.get(6)
    assert c6.ndims == 3 and c6.radius == 1 and len(c6.terms) == 7 and c6.model == 0
    assert np.float32(c6.terms[0][0]) == np.float32(1.0 - 6 * 0.15)      # 0.1, folded in double
    assert 6 * 0.15 < 1.0                                                   # explicit 3-D heat: kappa < 1/6
    c7 = CF.get(7)
    assert c7.model == 1 and c7.radius == 1 and len(c7.terms) == 7
    assert [float(x) for x in CF.fd2_weights(2)] == [-2.0, 1.0]
    assert c7.terms[0][0] == pytest.approx(-6.0) and c7.terms[1][0] == pytest.approx(1.0)
    assert c7.field == CF.get(3).field and c7.dt == pytest.approx(CF.get(3).dt)   # config 3's leapfrog
    bp6, bp7 = CF.BENCH_PLANS[6], CF.BENCH_PLANS[7]
    assert bp6["fused"] == 3 and bp7["fused"] == 3 and bp7["mode"] == "reference"


def test_host_buffer_checks_reject_wrong_dtype_and_layout():
    """upload / download / execute_host pass float* + element count: a
    float16, float64 or strided array must raise, not overrun."""
    import numpy as np
    from paper_1806_08299_b200 import tiler as T
    T._host_f32(np.zeros(8, np.float32), "download")
    for bad in (np.zeros(8, np.float16), np.zeros(8, np.float64), np.zeros(16, np.float32)[::2], [0.0] * 8):
        with pytest.raises(T.Error):
            T._host_f32(bad, "download")
    ro = np.zeros(8, np.float32)
    ro.flags.writeable = False
    T._host_f32(ro, "upload")
    with pytest.raises(T.Error):
        T._host_f32(ro, "download")
