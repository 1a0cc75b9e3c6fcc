"""CPU-side checks of the boundary: the C-ABI library builds, loads and exports every entry
point declared in include/gp.h, and the Python binding declares each of them. No GPU calls."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "gp.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:gp_status|const char\*|void)\s+(gp_\w+)\s*\(", src,
                                 flags=re.M)))


@pytest.fixture(scope="module")
def lib():
    from paper_2110_11226_b200 import build, _capi
    build.build()
    return ctypes.CDLL(_capi.LIB_PATH)


def test_header_declares_north_star_entry_points():
    d = _declared()
    for name in ("gp_evaluate", "gp_tournament_select", "gp_generation"):
        assert name in d
    assert len(d) >= 19


def test_library_exports_every_declared_symbol(lib):
    for name in _declared():
        assert hasattr(lib, name), name


def test_binding_declares_every_symbol():
    from paper_2110_11226_b200 import _capi
    assert set(_declared()) == set(_capi.SIGNATURES)


def test_struct_layouts_match_header(lib):
    from paper_2110_11226_b200 import _capi
    c = _capi.GpConfig()
    fn = getattr(lib, "gp_config_default")
    fn.argtypes = [ctypes.c_void_p]
    fn(ctypes.byref(c))
    # Table 6 defaults, read back through the ctypes layout
    assert c.population_size == 35 and c.tournament_size == 4
    assert abs(c.parsimony - 0.01) < 1e-9 and c.p_crossover == 0.7 and c.p_hoist == 0.05
    assert list(c.function_set[:c.n_functions]) == [2, 3, 4, 5, 9, 10, 11]
    assert c.stack_capacity == 20 and c.seed == 2110


def test_status_strings_and_no_gpu_calls(lib):
    fn = lib.gp_status_string
    fn.restype = ctypes.c_char_p
    fn.argtypes = [ctypes.c_int]
    assert fn(0) == b"GP_OK" and fn(3) == b"GP_ERR_UNSUPPORTED"
    v = lib.gp_version
    v.restype = ctypes.c_char_p
    assert b"sm_100a" in v()


def test_opcode_numbering_matches_oracle_interface():
    """gp.h's opcode enum is the interface the oracle retypes independently."""
    import oracle
    src = open(os.path.join(ROOT, "include", "gp.h")).read()
    enum = dict((m.group(1).lower(), int(m.group(2)))
                for m in re.finditer(r"GP_OP_(\w+)\s*=\s*(\d+)", src))
    for i, name in enumerate(oracle.NAMES):
        assert enum[name] == i, name
