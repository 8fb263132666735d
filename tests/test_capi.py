"""The C-ABI library builds for sm_100a, loads, and exports every header symbol (no GPU)."""
import ctypes
import subprocess

import pytest

from paper_2101_08431_b200 import _build, _lib


@pytest.fixture(scope="module")
def so_path():
    return _build.build()


def test_exports_every_header_symbol(so_path):
    so = ctypes.CDLL(so_path)
    names = _lib.header_symbols()
    assert len(names) >= 6
    missing = [n for n in names if not hasattr(so, n)]
    assert not missing, missing
    # every declared symbol has a ctypes signature in the binding
    assert set(names) <= set(_lib.SIGNATURES), set(names) - set(_lib.SIGNATURES)


def test_sass_is_sm100a(so_path):
    out = subprocess.run(["cuobjdump", "--list-elf", so_path], capture_output=True, text=True)
    assert out.returncode == 0
    assert "sm_100a" in out.stdout


def test_no_cpu_fallback_without_device(so_path, monkeypatch):
    import torch

    from paper_2101_08431_b200 import kernels
    from paper_2101_08431_b200.errors import NativeLibraryError

    monkeypatch.setattr(torch.cuda, "is_available", lambda: False)
    import numpy as np

    with pytest.raises(NativeLibraryError):
        kernels.block_cholesky(np.eye(2)[None])
