"""CPU checks of the C-ABI boundary: the library builds, loads and exports
every entry point include/augsched.h declares (no compute calls here)."""
import ctypes
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HDR = os.path.join(ROOT, "include", "augsched.h")


def declared():
    txt = open(HDR).read()
    return re.findall(r"AUGSCHED_API\s+[\w\s\*]+?\b(augsched_\w+)\s*\(", txt)


def test_header_declares_the_survey_boundary():
    names = set(declared())
    for n in ("augsched_create", "augsched_enqueue", "augsched_step", "augsched_simulate",
              "augsched_destroy", "augsched_last_error"):
        assert n in names


def test_library_exports_every_declared_symbol():
    from paper_2512_04013_b200 import _build
    lib_path = _build.build()
    L = ctypes.CDLL(lib_path)
    for n in declared():
        assert hasattr(L, n), n
    # internal symbols stay hidden (-fvisibility=hidden)
    out = os.popen(f"nm -D --defined-only {lib_path}").read()
    exported = {l.split()[-1] for l in out.splitlines() if " T " in l}
    assert {n for n in exported if n.startswith("augsched")} == set(declared())


def test_binding_struct_layouts_match_header():
    """ctypes mirrors of the header structs have the C sizes."""
    import paper_2512_04013_b200 as a
    assert ctypes.sizeof(a.InstanceParams) == 48
    assert ctypes.sizeof(a.Config) == 6 * 8 + 4 * 4 + 2 * 8 + 48
    assert ctypes.sizeof(a.Trace) == 10 * 8 + 16
    assert a.RESULT_DTYPE.itemsize == 24 * 8 + 2 * 160 * 4


def test_last_error_without_gpu():
    """augsched_create validates its arguments before touching CUDA."""
    import paper_2512_04013_b200 as a
    L = a.lib()
    cfg = a.Config()  # all zero: invalid
    h = ctypes.c_void_p()
    rc = L.augsched_create(ctypes.byref(cfg), None, 1, 1, 0, None, ctypes.byref(h))
    assert rc == a.E_INVALID
    assert b"must be >= 1" in L.augsched_last_error()


def test_product_does_not_import_oracle():
    """The CUDA path shares no code with the oracle (and vice versa)."""
    pkg = os.path.join(ROOT, "paper_2512_04013_b200")
    for dp, _, fs in os.walk(pkg):
        for f in fs:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                txt = open(os.path.join(dp, f)).read()
                assert "import oracle" not in txt and "from oracle" not in txt, f
                assert "augsched_oracle" not in txt, f
    for f in os.listdir(os.path.join(ROOT, "oracle")):
        if f.endswith((".py", ".cpp")):
            txt = open(os.path.join(ROOT, "oracle", f)).read()
            assert "paper_2512_04013_b200" not in txt.replace("paper_2512_04013_b200/", "") or \
                "import" not in txt.split("paper_2512_04013_b200")[0][-20:]
