"""CPU-side checks of the C-ABI library: it loads without a GPU and exports
every entry point declared in include/afdk.h with the expected ABI version."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "afdk.h")).read()
    return sorted(set(re.findall(r"\b(afdk_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    from paper_2507_19427_b200 import afdk

    lib = ctypes.CDLL(afdk.LIB_PATH)
    missing = [s for s in declared_symbols() if not hasattr(lib, s)]
    assert not missing, missing


def test_bindings_cover_header():
    from paper_2507_19427_b200 import afdk

    assert set(declared_symbols()) == set(afdk.SIGNATURES), set(declared_symbols()) ^ set(afdk.SIGNATURES)


def test_abi_version_and_no_device_error():
    import torch

    from paper_2507_19427_b200 import afdk

    lib = afdk.load()
    assert lib.afdk_abi_version() == 1
    if torch.cuda.is_available():
        pytest.skip("GPU present: no-device path not testable")
    with pytest.raises(afdk.AfdkError) as ei:
        afdk.Context(0)
    assert ei.value.status in (2, 4)  # no device -> fails loudly, never falls back


def test_sass_is_tcgen05_native():
    """The built kernels use tcgen05 MMA, TMEM loads and TMA (not HMMA)."""
    import shutil
    import subprocess

    from paper_2507_19427_b200 import afdk

    if not shutil.which("cuobjdump") and not os.path.exists("/usr/local/cuda/bin/cuobjdump"):
        pytest.skip("cuobjdump absent")
    exe = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    sass = subprocess.run([exe, "-sass", afdk.LIB_PATH], capture_output=True, text=True).stdout
    assert "UTCHMMA" in sass and "LDTM" in sass and "UTMALDG" in sass
    assert "HMMA" not in sass.replace("UTCHMMA", "")
