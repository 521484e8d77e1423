"""User vertex programs (include/ipregel.h "user vertex programs", csrc/program.cuh): host-side
checks that need no GPU -- NVRTC compiles every catalogued program for sm_100a, compile errors
and bad descriptors are reported through the C ABI."""
import pytest

import paper_2010_08781_b200 as ipr
from paper_2010_08781_b200 import programs


@pytest.mark.parametrize("name", sorted(programs.CATALOG))
def test_catalog_programs_compile(name):
    p = programs.compile(name)
    assert p.cubin_bytes > 10000
    assert "error" not in p.log.lower()
    p.close()


def test_compile_error_is_reported_with_the_log():
    bad = programs.SSSP.replace("return ipr_sat_add(message, weight);", "return undefined_fn(message);")
    with pytest.raises(ipr.IpregelError) as e:
        ipr.Program(bad, "u32", "min")
    assert e.value.status == ipr.ERR_INVALID_ARGUMENT
    assert "undefined_fn" in str(e.value)
    assert "user_program.cu" in str(e.value)     # errors point at the user's own source lines


def test_missing_entry_point_is_a_compile_error():
    src = programs.HASHMIN_CC.split("__device__ unsigned ipr_edge")[0]
    with pytest.raises(ipr.IpregelError) as e:
        ipr.Program(src, "u32", "min", symmetric=True)
    assert e.value.status == ipr.ERR_INVALID_ARGUMENT
    assert "ipr_edge" in str(e.value)


def test_bad_descriptors():
    import ctypes
    lib = ipr.load()
    for vt, comb, sym, res in ((7, 1, 0, 0), (0, 9, 0, 0), (0, 1, 2, 0), (0, 1, 0, 1)):
        d = ipr.ipregel.ProgramDesc()
        src = programs.SSSP.encode()
        d.source, d.value_type, d.combiner, d.symmetric, d.reserved = src, vt, comb, sym, res
        h = ctypes.c_void_p()
        assert lib.ipregel_program_create(ctypes.byref(d), ctypes.byref(h)) == ipr.ERR_INVALID_ARGUMENT
        assert not h.value
    assert lib.ipregel_program_create(None, ctypes.byref(ctypes.c_void_p())) == ipr.ERR_INVALID_ARGUMENT


def test_value_type_must_match_the_source():
    # the f64 PageRank source as a u32 program: ipr_init's signature no longer matches
    with pytest.raises(ipr.IpregelError):
        ipr.Program(programs.PAGERANK, "u32", "sum")
