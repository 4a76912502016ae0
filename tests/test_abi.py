"""The C-ABI library builds, loads and exports every symbol include/dawnpiper.h
declares (no device needed; nothing here launches a kernel)."""
import re
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent


def _declared():
    text = (ROOT / "include" / "dawnpiper.h").read_text()
    return sorted(set(re.findall(r"\b(dpn_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_the_abi():
    names = _declared()
    for must in ("dpn_gemm", "dpn_swap_out", "dpn_swap_in", "dpn_p2p_copy", "dpn_layernorm_fwd",
                 "dpn_xent", "dpn_adamw", "dpn_last_error", "dpn_init"):
        assert must in names


def test_library_exports_every_declared_symbol():
    from paper_2505_05856_b200.build import build
    from paper_2505_05856_b200 import _lib
    build()
    lib = _lib.load_library()
    missing = [n for n in _declared() if not hasattr(lib, n)]
    assert not missing, missing
    assert lib.dpn_version() == 1
    # every declared symbol is typed by the binding
    assert set(_declared()) <= set(_lib.SIGNATURES) | {"dpn_last_error", "dpn_arena_malloc",
                                                      "dpn_arena_free"}


def test_bad_arguments_fail_with_a_message():
    import ctypes
    from paper_2505_05856_b200 import _lib
    lib = _lib.load_library()
    rc = lib.dpn_gemm(None, None)
    assert rc == 1
    assert b"null args" in lib.dpn_last_error()
    g = _lib.GemmArgs()
    g.M, g.N, g.K = 0, 8, 8
    assert lib.dpn_gemm(ctypes.byref(g), None) == 1
    assert b"positive" in lib.dpn_last_error()


def test_missing_extension_fails_loudly(monkeypatch, tmp_path):
    from paper_2505_05856_b200 import _lib
    monkeypatch.setattr(_lib, "_lib", None)
    monkeypatch.setattr(_lib, "SO_PATH", tmp_path / "nope.so")
    with pytest.raises(_lib.DpnError, match="not built"):
        _lib.load_library()
