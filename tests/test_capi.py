"""CPU-side checks of the drop-in boundary: the C-ABI library loads and
exports every function include/combo_cuda.h declares; the ctypes mirror
covers them all. No compute calls (no GPU here)."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "combo_cuda.h")
LIB = os.path.join(ROOT, "paper_2204_13624_b200", "libcombo_cuda.so")


def declared():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(combo_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_entry_points():
    names = declared()
    for n in ["combo_ctx_create", "combo_solve", "combo_stress_sweep", "combo_project", "combo_coarsen",
              "combo_normals", "combo_bind_materials", "combo_tangent_matvec", "combo_dfmg_stress"]:
        assert n in names


@pytest.mark.skipif(not os.path.exists(LIB), reason="library not built")
def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(LIB)
    missing = [n for n in declared() if not hasattr(lib, n)]
    assert not missing, missing


def test_ctypes_mirror_covers_header():
    from paper_2204_13624_b200.combo import SIGNATURES

    missing = [n for n in declared() if n not in SIGNATURES]
    assert not missing, missing


def build_dropin_example(out):
    import subprocess

    src = os.path.join(ROOT, "tests", "cpp", "dropin_example.cpp")
    libdir = os.path.dirname(LIB)
    subprocess.run(["g++", "-std=c++17", "-O2", "-Wall", "-Wextra", "-I", os.path.join(ROOT, "include"), src,
                    "-L", libdir, "-lcombo_cuda", f"-Wl,-rpath,{libdir}", "-o", out], check=True)
    return out


@pytest.mark.skipif(not os.path.exists(LIB), reason="library not built")
def test_cpp_dropin_layer_compiles_and_links(tmp_path):
    exe = build_dropin_example(str(tmp_path / "dropin"))
    assert os.path.exists(exe)


@pytest.mark.skipif(not os.path.exists(LIB), reason="library not built")
def test_version_and_error_paths_without_gpu():
    lib = ctypes.CDLL(LIB)
    lib.combo_version.restype = ctypes.c_char_p
    assert b"sm_100a" in lib.combo_version()
    # null out-pointer is rejected with BadArgument (-13), never a crash
    lib.combo_ctx_create.argtypes = [ctypes.c_int, ctypes.c_void_p]
    assert lib.combo_ctx_create(0, None) == -13
    lib.combo_report_free.argtypes = [ctypes.c_void_p]
    assert lib.combo_report_free(None) == 0
