"""CPU checks of the boundary: libfj.so loads and exports every entry point include/fj.h declares
(no compute calls: there is no GPU here)."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _strip_c_comments(txt):
    """Drop /* */ blocks (across lines) and // line comments (to the end of their line only)."""
    return re.sub(r"//[^\n]*", "", re.sub(r"/\*.*?\*/", "", txt, flags=re.S))


def declared_functions():
    src = open(os.path.join(ROOT, "include", "fj.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(fj_[a-z_0-9]+)\s*\(", src)))


def test_header_declares_the_survey_boundary():
    names = set(declared_functions())
    for required in ["fj_csr_from_edges", "fj_graph_create", "fj_graph_info", "fj_graph_degrees", "fj_apply",
                     "fj_solve", "fj_quantities", "fj_approxim", "fj_graph_destroy", "fj_status_str",
                     "fj_last_error", "fj_opinion_stats", "fj_approxim_host", "fj_set_allocator"]:
        assert required in names


def test_library_exports_every_declared_symbol():
    from paper_2101_08143_b200 import build as B
    so = B.build()
    lib = ctypes.CDLL(so)
    missing = [f for f in declared_functions() if not hasattr(lib, f)]
    assert not missing, missing
    lib.fj_abi_version.restype = ctypes.c_int
    assert lib.fj_abi_version() == 1
    lib.fj_status_str.restype = ctypes.c_char_p
    assert lib.fj_status_str(6) == b"FJ_E_NO_CONVERGENCE"


def test_invalid_arguments_fail_without_gpu():
    """Argument validation happens before any device call."""
    import paper_2101_08143_b200 as fj
    L = fj.lib()
    h = ctypes.c_void_p()
    st = L.fj_graph_create(0, 0, None, None, None, 0, 1, None, ctypes.byref(h))
    assert st == 1 and not h.value
    assert b"n must be" in L.fj_last_error()
    assert L.fj_solve(None, 1, None, None, None, None, None) == 1


def test_set_allocator_argument_rules_without_gpu():
    """fj_set_allocator: alloc and free both set or both NULL (no device call involved)."""
    import paper_2101_08143_b200 as fj
    from paper_2101_08143_b200 import binding as b
    L = fj.lib()
    a = b._ALLOC_FN(lambda n, s, c: None)
    null_free = ctypes.cast(None, b._FREE_FN)
    assert L.fj_set_allocator(a, null_free, None) == 1
    assert b"both" in L.fj_last_error()
    assert L.fj_set_allocator(ctypes.cast(None, b._ALLOC_FN), null_free, None) == 0
    assert fj.allocator_live_blocks() == 0


def test_device_frees_go_through_the_allocator_hook():
    """Workspace memory may come from a caller allocator (fj_set_allocator): only graph.cu's
    dfree_on may call cudaFreeAsync (a raw free of a torch block would release its whole segment)."""
    csrc = os.path.join(ROOT, "paper_2101_08143_b200", "csrc")
    for f in os.listdir(csrc):
        code = _strip_c_comments(open(os.path.join(csrc, f)).read())
        n = len(re.findall(r"\bcudaFreeAsync\s*\(", code))
        assert n == (1 if f == "graph.cu" else 0), (f, n)


def test_product_path_does_not_import_oracle():
    pkg = os.path.join(ROOT, "paper_2101_08143_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                txt = open(os.path.join(dirpath, f)).read()
                code = _strip_c_comments(txt) if not f.endswith(".py") else re.sub(r"#.*", "", txt)
                assert "oracle" not in code.lower(), f


def test_missing_library_raises(tmp_path):
    from paper_2101_08143_b200 import binding
    with pytest.raises(ImportError):
        binding._lib_backup = binding._lib
        binding._lib = None
        try:
            binding.load_library(str(tmp_path / "nope.so"))
        finally:
            binding._lib = binding._lib_backup


def test_alg1_delta_host_arithmetic_matches_oracle():
    """fj_alg1_delta is host-only arithmetic (Algorithm 1 line 1; clamp S:L153; residual map):
    it must agree with the oracle's independent transcription on a range of graph sizes."""
    import oracle as O
    import paper_2101_08143_b200 as fj
    cases = [(1, 0.0, 0.0, 0.0, 1.0, 0.1), (2, 1.0, 1.0, 1.0, 0.5 ** 0.5, 1e-6), (2000, 1.0, 1.0, 90.0, 12.9, 1e-6),
             (300, 0.2, 3.0, 40.0, 5.0, 0.25), (4_000_000, 1.0, 1.0, 9507.0, 577.0, 1e-6)]
    for c in cases:
        got = fj.alg1_delta(*c)
        want = O.alg1_delta(*c)
        for a, b in zip(got, want):
            assert a == pytest.approx(b, rel=1e-14), (c, got, want)
