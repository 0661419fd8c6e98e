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
