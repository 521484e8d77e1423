"""The C-ABI library loads and exports every symbol include/ipregel.h declares; host-only
entry points (no GPU needed) behave as documented."""
import ctypes
import os
import re

import numpy as np
import pytest

import paper_2010_08781_b200 as ipr

HEADER = os.path.join(os.path.dirname(__file__), "..", "include", "ipregel.h")


def declared_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(ipregel_[a-z_]+)\s*\(", text)))


def test_header_and_binding_agree():
    assert declared_functions() == sorted(ipr.ipregel.EXPORTS)


def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(ipr.ipregel.LIB_PATH)
    for name in declared_functions():
        assert hasattr(lib, name), name


def test_library_is_sm100a_only():
    out = os.popen(f"cuobjdump --list-elf {ipr.ipregel.LIB_PATH} 2>&1").read()
    assert "sm_100a" in out
    assert re.search(r"sm_(?!100a)\d+", out.replace("sm_100a", "")) is None


def test_status_strings_and_version():
    assert ipr.status_string(ipr.OK) == "IPREGEL_OK"
    assert ipr.status_string(ipr.ERR_MAX_SUPERSTEPS) == "IPREGEL_ERR_MAX_SUPERSTEPS"
    assert ipr.load().ipregel_abi_version() == 1


def test_run_params_default():
    p = ipr.run_params_default()
    assert (p.mode, p.pagerank_iterations, p.sssp_source, p.flags) == (ipr.MODE_AUTO, 10, 0, 0)
    assert abs(p.push_fraction - 0.04) < 1e-7
    assert p.pagerank_tolerance == -1.0


def test_struct_layouts_match_header(tmp_path):
    """sizeof/offsetof of every ABI struct from the C compiler equal the ctypes binding's."""
    import subprocess
    structs = {"ipregel_graph_desc": ipr.ipregel.GraphDesc, "ipregel_run_params": ipr.RunParams,
               "ipregel_stats": ipr.ipregel.Stats, "ipregel_program_desc": ipr.ipregel.ProgramDesc}
    lines = ['#include <stdio.h>', '#include <stddef.h>', f'#include "{os.path.abspath(HEADER)}"',
             "int main(void) {"]
    for cname, cls in structs.items():
        lines.append(f'printf("%zu\\n", sizeof({cname}));')
        for fname, _ in cls._fields_:
            lines.append(f'printf("%zu\\n", offsetof({cname}, {fname}));')
    lines.append("return 0; }")
    src = tmp_path / "layout.c"
    src.write_text("\n".join(lines))
    exe = tmp_path / "layout"
    subprocess.check_call(["gcc", "-o", str(exe), str(src)])
    got = [int(x) for x in subprocess.check_output([str(exe)]).split()]
    want = []
    for cls in structs.values():
        want.append(ctypes.sizeof(cls))
        want += [getattr(cls, f).offset for f, _ in cls._fields_]
    assert got == want


def test_partition_edge_balanced():
    # cost prefix of 10 vertices with a hub at vertex 3
    cost = np.array([1, 1, 1, 50, 1, 1, 1, 1, 1, 1], np.int64)
    cp = np.concatenate([[0], np.cumsum(cost)])
    b = ipr.partition(cp, 2)
    assert b[0] == 0 and b[-1] == 10
    assert np.all(np.diff(b) >= 0)
    # the first range must end right after the hub reaches half the total cost
    half = cp[-1] / 2
    assert cp[b[1]] >= half and cp[b[1] - 1] < half
    b8 = ipr.partition(cp, 8)
    assert len(b8) == 9 and np.all(np.diff(b8) >= 0)
    # deterministic
    np.testing.assert_array_equal(b8, ipr.partition(cp, 8))


def test_partition_rejects_bad_prefix():
    with pytest.raises(ipr.IpregelError):
        ipr.partition(np.array([0, 5, 3]), 2)
    with pytest.raises(ipr.IpregelError):
        ipr.partition(np.array([1, 5]), 2)


def test_library_fails_loudly_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    st = ipr.load().ipregel_device_check(0)
    assert st in (ipr.ERR_CUDA, ipr.ERR_UNSUPPORTED)
    assert ipr.last_error()


def test_product_path_never_imports_the_oracle():
    """The oracle is test infrastructure: the package (and its program catalog) must not import
    it, and no product, input-generator or tool source mentions it as a module (only tests/,
    smoke() and bench.py's cpu_baseline / --impl reference legs use it)."""
    import subprocess
    import sys
    code = ("import sys; import paper_2010_08781_b200, paper_2010_08781_b200.programs; "
            "print('oracle' in sys.modules)")
    out = subprocess.check_output([sys.executable, "-c", code],
                                  cwd=os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    assert out.decode().strip() == "False"
    repo = os.path.join(os.path.dirname(__file__), "..")
    pkg = os.path.join(repo, "paper_2010_08781_b200")
    for root, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                text = open(os.path.join(root, f)).read()
                assert "import oracle" not in text and "oracle/" not in text, f
    # tools, input generators and the header: no import, include or link of the oracle
    uses = ("import oracle", "from oracle", "include \"oracle", "include \"../oracle", "liboracle")
    for sub in ("tools", "inputs", "include"):
        for root, _, files in os.walk(os.path.join(repo, sub)):
            for f in files:
                if f.endswith((".py", ".cu", ".cuh", ".h", ".c")):
                    text = open(os.path.join(root, f)).read()
                    assert not any(u in text for u in uses), f
