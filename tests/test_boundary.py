"""The C-ABI library loads and exports every symbol include/rpd.h declares (-m "not gpu":
no compute calls)."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_functions():
    src = open(os.path.join(ROOT, "include", "rpd.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(rpd_[a-z_]+)\s*\(", src)))


def test_header_declares_the_boundary():
    names = declared_functions()
    for f in ("rpd_relations", "rpd_clip", "rpd_update_partial", "rpd_create", "rpd_destroy",
              "rpd_last_error"):
        assert f in names


def test_library_builds_and_exports_all_symbols():
    import paper_2403_18761_b200 as P
    path = P.build()
    lib = ctypes.CDLL(path)
    for f in declared_functions():
        assert hasattr(lib, f), f"{f} declared in rpd.h but not exported"
    assert set(P.EXPORTED) == set(declared_functions())
    lib.rpd_version.restype = ctypes.c_char_p
    assert b"sm_100a" in lib.rpd_version()


def test_library_is_sm100a():
    import subprocess
    import paper_2403_18761_b200 as P
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", P.build()],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_null_ctx_is_einval():
    import paper_2403_18761_b200 as P
    L = P.load_library()
    assert L.rpd_set_option(None, 1, 0) == -1
    assert L.rpd_clip(None, None) == -1
    assert L.rpd_last_error(None) == b"null rpd_ctx"
