"""CPU-side checks of the C-ABI boundary: libhata.so builds, loads and exports
every symbol include/hata.h declares; host-side validation rejects bad
arguments synchronously without touching a device."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "hata.h")


@pytest.fixture(scope="module")
def lib():
    from paper_2506_02572_b200 import build, _lib
    build.build()
    return _lib.load()


def declared_symbols():
    txt = open(HEADER).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(hata_[a-z_0-9]+)\s*\(", txt)))


def test_header_symbols_exported(lib):
    from paper_2506_02572_b200 import _lib
    syms = declared_symbols()
    assert len(syms) >= 12
    out = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\bT (hata_\w+)", out))
    for s in syms:
        assert s in exported, s
        assert hasattr(lib, s)
    assert set(_lib.EXPORTS) == set(syms)


def test_status_strings_and_version(lib):
    assert lib.hata_status_string(0) == b"HATA_OK"
    assert lib.hata_status_string(1) == b"HATA_ERR_INVALID_ARG"
    assert lib.hata_status_string(4) == b"HATA_ERR_WORKSPACE"
    assert b"sm_100a" in lib.hata_version()


def test_validation_rejects_before_launch(lib):
    from paper_2506_02572_b200._lib import Strides
    s = Strides(0, 0, 0)
    P = ctypes.c_void_p(4096)  # never dereferenced: validation fails first
    # k < 1
    assert lib.hata_decode_topk_attn(P, P, P, s, 1, P, s, P, 1, 32, 8, 128, 128, P, 100, 0, 0.0, P, 0,
                                     None, None, None, None, 0, None) == 1
    # H_q % H_kv != 0
    assert lib.hata_decode_topk_attn(P, P, P, s, 1, P, s, P, 1, 30, 8, 128, 128, P, 100, 4, 0.0, P, 0,
                                     None, None, None, None, 0, None) == 1
    # rbits % 32 != 0
    assert lib.hata_hash_keys(P, Strides(1, 1, 128), 1, P, 1, 1, 128, 100, 0, 10, 16, P, Strides(1, 1, 4), None) == 1
    # unsupported head dim
    assert lib.hata_hash_keys(P, Strides(1, 1, 64), 1, P, 1, 1, 64, 128, 0, 10, 16, P, Strides(1, 1, 4), None) == 2
    # t0 + n beyond the capacity
    assert lib.hata_hash_keys(P, Strides(1, 1, 128), 1, P, 1, 1, 128, 128, 8, 10, 16, P, Strides(1, 1, 4), None) == 3
    # unknown option; known options accepted
    assert lib.hata_set_option(7, 1) == 1
    assert lib.hata_set_option(0, 1) == 0 and lib.hata_set_option(1, 1) == 0 and lib.hata_set_option(2, 1) == 0
    # null pointers
    assert lib.hata_append(None, P, 1, P, P, P, s, P, s, P, 10, 1, 1, 128, 128, None) == 1
    assert lib.hata_shard_combine(None, 2, 1, 32, 128, P, 0, None) == 1


def test_workspace_query(lib):
    from paper_2506_02572_b200 import decode_ranks, decode_workspace_size
    # CFG-4: 8 (b, g) units x M=18 ranks on a 148-SM part; the ranks exchange
    # prefix counts of their histograms (513 bins + 1) and flash-decoding
    # partials (G heads x (d + 2) floats) through the workspace
    M = decode_ranks(1, 32, 8, 128, 128, 131072, 2048)
    assert M == 18
    ws = decode_workspace_size(1, 32, 8, 128, 128, 131072, 2048)
    assert ws >= 8 * M * (514 * 4 + 4 * 130 * 4)
    # one rank per unit (128 units): no exchange; D of a 128K chunk spills to the workspace
    assert decode_ranks(16, 32, 8, 128, 128, 131072, 2048) == 1
    assert decode_workspace_size(16, 32, 8, 128, 128, 131072, 2048) >= 128 * 131072 * 2
    assert decode_workspace_size(1, 32, 8, 128, 100, 1000, 10) == 0  # invalid -> 0


def test_product_library_reads_no_debug_env(lib):
    """The diagnostics knobs (rank count, debug bits) live only in the
    diagnostics build; the product library reads no HATA_* environment."""
    from paper_2506_02572_b200 import _lib
    data = open(_lib.LIB_PATH, "rb").read()
    for knob in (b"HATA_RANKS", b"HATA_DEBUG", b"HATA_HINT", b"HATA_PDL"):
        assert knob not in data, knob
