"""The C-ABI library loads and exports every entry point include/defmm_b200.h
declares (no compute calls: this runs without a GPU)."""

import ctypes
import os
import re

from conftest import ROOT
from paper_2202_04894_b200 import _lib


def _declared():
    """Every entry point the header declares (typed families expanded)."""
    src = open(os.path.join(ROOT, "include", "defmm_b200.h")).read()
    names = set(re.findall(r"\b(defmm_[a-z0-9_]+)\s*\(", src))
    typed = {n for n in names if n.endswith("##SUFFIX")} | set(re.findall(r"\b(defmm_[a-z0-9_]+)_##SUFFIX", src))
    names = {n for n in names if "##" not in n and n != "defmm_tree"}
    for suffix in re.findall(r"^DEFMM_DECLARE_TYPED\((\w+)\)", src, re.M):
        names |= {f"{t}_{suffix}" for t in typed if "##" not in t}
    return sorted(names)


def test_header_and_binding_agree():
    assert sorted(_lib.EXPORTED) == _declared()


def test_library_exports_every_symbol():
    lib = ctypes.CDLL(_lib.LIB_PATH)
    for name in _declared():
        assert hasattr(lib, name), name
    assert _lib.load().defmm_abi_version() == 1


def test_library_is_sm100a():
    import subprocess

    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", _lib.LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out
