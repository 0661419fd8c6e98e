"""CPU-side checks of the C-ABI boundary: the library builds for sm_100a, loads
without a GPU, and exports every symbol include/dmf.h declares."""
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "dmf.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(dmf_[a-z_]+)\s*\(", src)))


def test_header_declares_north_star_entry_points():
    names = _declared()
    for f in ("dmf_create", "dmf_static_solve", "dmf_apply_batch", "dmf_flow_value", "dmf_min_cut_source_side"):
        assert f in names


def test_library_loads_and_exports_all_symbols():
    from paper_2511_05895_b200 import build, load_library
    build.build()
    L = load_library()
    for name in _declared():
        assert hasattr(L, name), name
    out = subprocess.run(["nm", "-D", "--defined-only", build.LIB], capture_output=True, text=True).stdout
    for name in _declared():
        assert re.search(r"\bT " + name + r"\b", out), name


def test_library_is_sm100a():
    from paper_2511_05895_b200 import build
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", build.LIB], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_no_oracle_import_in_product():
    pkg = os.path.join(ROOT, "paper_2511_05895_b200")
    for dp, _, fs in os.walk(pkg):
        for f in fs:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                txt = open(os.path.join(dp, f)).read()
                assert "import oracle" not in txt and "from oracle" not in txt and "oracle.c" not in txt, f


def test_ctypes_structs_match_the_c_header(tmp_path):
    """The binding's ctypes mirrors of dmf_options / dmf_stats have the C layout
    (size and every field offset), compiled here with gcc from include/dmf.h."""
    import ctypes
    import paper_2511_05895_b200 as P
    lines = ['#include <stdio.h>', '#include <stddef.h>', '#include "dmf.h"', 'int main(void) {']
    for cname, cls in (("dmf_options", P.Options), ("dmf_stats", P.Stats)):
        lines.append(f'printf("{cname} sizeof %zu\\n", sizeof({cname}));')
        for f, _ in cls._fields_:
            lines.append(f'printf("{cname} {f} %zu\\n", offsetof({cname}, {f}));')
    lines.append("return 0; }")
    src = tmp_path / "abi.c"
    src.write_text("\n".join(lines))
    exe = tmp_path / "abi"
    subprocess.check_call(["gcc", "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe)])
    out = subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout.split("\n")
    got = {(a, b): int(c) for a, b, c in (l.split() for l in out if l)}
    for cname, cls in (("dmf_options", P.Options), ("dmf_stats", P.Stats)):
        assert got[(cname, "sizeof")] == ctypes.sizeof(cls), cname
        for f, _ in cls._fields_:
            assert got[(cname, f)] == getattr(cls, f).offset, (cname, f)


def test_binding_rejects_mismatched_batches_without_a_gpu():
    """Argument marshalling errors are raised before any library call."""
    import numpy as np
    import paper_2511_05895_b200 as P
    f = P.DynMaxFlow.__new__(P.DynMaxFlow)     # no handle: the checks must fire first
    with pytest.raises(ValueError):
        f.apply_batch(np.zeros(3, np.int32), np.zeros(2, np.int32), np.zeros(3, np.int32))
    with pytest.raises(ValueError):
        f.apply_batch(np.zeros((2, 2), np.int32), np.zeros(4, np.int32), np.zeros(4, np.int32))
