"""CPU-side checks of the C ABI: the library builds/loads and exports every symbol that
include/tt_b200.h declares; host-only entry points behave without a GPU."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "tt_b200.h")


def _declared():
    txt = open(HEADER).read()
    return sorted(set(re.findall(r"^TT_API\s+[\w\s\*]+?\b(tt_\w+)\(", txt, flags=re.M)))


@pytest.fixture(scope="module")
def lib():
    from paper_2211_08770_b200 import _build, _native
    _build.build_library()
    return _native.load()


def test_header_declares_entry_points():
    names = _declared()
    for must in ("tt_round", "tt_round_batch", "tt_dot_batch", "tt_gram", "tt_gram_blocks", "tt_sum",
                 "tt_axpy", "tt_element", "tt_orth", "tt_ctx_create"):
        assert must in names


def test_library_exports_every_declared_symbol(lib):
    from paper_2211_08770_b200 import _native
    names = _declared()
    assert names == sorted(_native.EXPORTED)
    for name in names:
        assert hasattr(lib, name), name


def test_only_abi_symbols_are_exported(lib):
    out = os.popen(f"nm -D --defined-only {lib._name}").read()
    syms = [ln.split()[-1] for ln in out.splitlines() if " T " in ln]
    assert sorted(s for s in syms if s.startswith("tt_")) == _declared()


def test_host_only_calls(lib):
    assert lib.tt_status_string(0) == b"TT_OK"
    assert lib.tt_status_string(7) == b"TT_ESINGULAR_GRAM"
    assert lib.tt_last_error(None) == b"null context"
    assert lib.tt_ctx_launch_count(None) == -1
    assert lib.tt_ctx_destroy(None) == 1  # TT_EINVAL


def test_ctx_create_without_gpu_fails_cleanly(lib):
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    h = ctypes.c_void_p()
    st = lib.tt_ctx_create(0, None, ctypes.byref(h))
    assert st != 0 and not h.value


def test_product_path_has_no_oracle_import():
    pkg = os.path.join(ROOT, "paper_2211_08770_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith(".py"):
                src = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in src and "from oracle" not in src, f
