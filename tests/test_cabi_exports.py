"""The C-ABI library loads without a GPU and exports every entry point include/*.h declares."""
import ctypes
import os
import re

from paper_2211_14969_b200 import leaf_gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


LIBS = {"hps_leaf_gpu.h": lambda: leaf_gpu.LIB_PATH,
        "hps_slablu.h": lambda: os.path.join(ROOT, "paper_2211_14969_b200", "_lib", "libhps_slablu_b200.so")}


def declared_functions(header):
    src = open(os.path.join(ROOT, "include", header)).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return set(re.findall(r"\b(hps_\w+)\s*\(", src))


def test_every_header_has_a_library():
    assert sorted(f for f in os.listdir(os.path.join(ROOT, "include")) if f.endswith(".h")) == sorted(LIBS)


def test_library_exports_every_declared_symbol():
    for header, path in LIBS.items():
        lib = ctypes.CDLL(path())
        decl = declared_functions(header)
        assert len(decl) >= 5, header
        missing = [n for n in sorted(decl) if not hasattr(lib, n)]
        assert not missing, (header, missing)
    assert set(leaf_gpu.EXPORTED) <= declared_functions("hps_leaf_gpu.h")


def test_version_string_without_gpu():
    assert b"sm_100a" in leaf_gpu.lib().hps_gpu_version()


def test_kernels_are_sm100a_dmma():
    """The shipped cubin is sm_100a and the LU kernel issues DMMA (FP64 tensor) instructions."""
    import shutil
    import subprocess
    if not shutil.which("cuobjdump"):
        return
    out = subprocess.run(["cuobjdump", "-sass", leaf_gpu.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    lu = out[out.find("k2_lu_schur_kernel"):]
    assert "DMMA.8x8x4" in lu
