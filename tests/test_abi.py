"""The C-ABI library loads without a GPU and exports exactly what include/sentinel_b200.h declares.

No compute call is made here (there is no GPU in the build container); argument
validation that happens before any CUDA call is exercised through the ABI.
"""

import ctypes
import re
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
HEADER = ROOT / "include" / "sentinel_b200.h"


@pytest.fixture(scope="module")
def lib():
    from paper_2510_00554_b200 import _native

    return _native.load()


def declared_functions():
    text = re.sub(r"/\*.*?\*/", "", HEADER.read_text(), flags=re.S)
    return sorted(set(re.findall(r"\b(snt_[a-z0-9_]+)\s*\(", text)))


def test_every_declared_symbol_is_exported_and_bound(lib):
    from paper_2510_00554_b200 import _native

    names = declared_functions()
    assert len(names) >= 17
    for name in names:
        assert hasattr(lib, name), f"{name} declared in the header but not exported"
    assert sorted(_native.SIGNATURES) == names, "ctypes signatures and header out of sync"


def test_header_cites_the_reference_interface():
    text = HEADER.read_text()
    for cite in ("merkle.py:93-114", "merkle.py:117-149", "merkle.py:152-165", "model.py:137-146",
                 "model.py:298-310", "dataset.py:41-49", "lattice.py:104-119", "errors.py"):
        assert cite in text


def test_constants_and_strings(lib):
    assert lib.snt_abi_version() == 3
    assert [lib.snt_digest_len(a) for a in (0, 1, 2, 3)] == [32, 64, 32, 0]
    assert lib.snt_strerror(0) == b"ok"
    assert b"invalid input" in lib.snt_strerror(-1)
    assert b"unknown" in lib.snt_strerror(-99)
    # workspace = ping-pong levels of the multi-launch reducer + counters, stage nodes and parked chain
    # states of the fused kernel; sized from (alg, count) alone, no device needed
    assert lib.snt_merkle_work_bytes(0, 79672) >= 2 * (78 + 1) * 32 + 4 * (79672 // 32)
    assert lib.snt_merkle_work_bytes(0, 799954) >= 2 * (99995 + 1) * 32 + 4 * (799954 // 32)
    assert lib.snt_merkle_work_bytes(0, 799954) > lib.snt_merkle_work_bytes(0, 79672) > lib.snt_merkle_work_bytes(0, 1) > 0
    assert lib.snt_merkle_work_bytes(1, 1000) > lib.snt_merkle_work_bytes(0, 1000)      # 64-byte digests, 16-word states
    assert lib.snt_merkle_work_bytes(7, 1000) == 0
    assert lib.snt_merkle_work_init(None, 0, None) == -1


def test_argument_validation_before_any_cuda_call(lib):
    handle = ctypes.c_void_p()
    ptrs = (ctypes.c_void_p * 1)(0x1000)
    sizes = (ctypes.c_uint64 * 1)(100)
    for bad_bs in (0, 63, 100, 8191):                        # model.py:93-95 -> ConfigError
        assert lib.snt_model_plan_create(ptrs, sizes, 1, bad_bs, None, ctypes.byref(handle)) == -3
    assert lib.snt_model_plan_create(ptrs, sizes, 0, 8192, None, ctypes.byref(handle)) == -1    # no tensors
    sizes[0] = 0
    assert lib.snt_model_plan_create(ptrs, sizes, 1, 8192, None, ctypes.byref(handle)) == -1    # zero bytes (model.py:166)
    assert not handle.value
    assert lib.snt_hash_blocks(0, None, None, None, 0, None, None) == -1                  # merkle.py:100-101
    assert lib.snt_hash_blocks(7, None, None, None, 1, None, None) == -3
    assert lib.snt_merkle_root(0, None, 0, None, 0, None, None) == -1                     # merkle.py:156-157
    assert lib.snt_merkle_inplace(None, 0, 0, 1, 0, None, None, 0, None, None) == -1
    assert lib.snt_lthash_samples(None, None, None, None, None, 0, 0, None, None, None, None, None) == -1
    assert lib.snt_lt_reduce(None, 0, None, None) == -1


def test_status_codes_map_to_reference_exceptions():
    from paper_2510_00554_b200 import errors

    pairs = {-1: errors.InvalidInput, -2: errors.InvalidState, -3: errors.ConfigError,
             -4: errors.ValidationError, -5: errors.ResourceError}
    for code, exc in pairs.items():
        with pytest.raises(exc):
            errors.raise_for_status(code, "x")
    errors.raise_for_status(0, "x")
    for cls in pairs.values():
        assert issubclass(cls, errors.SentinelError)


def test_product_never_imports_the_oracle():
    pkg = ROOT / "paper_2510_00554_b200"
    for py in pkg.rglob("*.py"):
        text = py.read_text()
        assert "sentinel_oracle" not in text and "c_oracle" not in text and "liboracle" not in text \
            or py.name == "build.py", f"{py} references the oracle"
    for src in (pkg / "csrc").glob("*"):
        assert "oracle" not in src.read_text()
