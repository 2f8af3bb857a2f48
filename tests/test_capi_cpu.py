"""C-ABI library checks that need no GPU: it loads, exports every symbol the
header declares, refuses to run without a device (no CPU fallback), and its
host-side generators are bit-identical to the oracle's."""
import ctypes as C
import os
import re

import numpy as np
import pytest

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
HEADER = os.path.join(ROOT, "include", "hetm_b200", "capi.h")


def declared_symbols():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(hetm_[a-z0-9_]+)\s*\(", src)))


def test_header_symbols_exported(hetm):
    lib = C.CDLL(hetm.LIB_PATH)
    names = declared_symbols()
    assert len(names) >= 40
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, f"capi.h declares but libhetm_b200.so does not export: {missing}"
    # and the Python binding covers all of them
    assert set(names) <= set(hetm.EXPORTED) | {"hetm_dev_config_default"}


def test_library_is_sm100a_only(hetm):
    """The fatbin carries sm_100a SASS (no PTX JIT fallback, no other arch)."""
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", hetm.LIB_PATH], capture_output=True, text=True).stdout
    archs = set(re.findall(r"sm_(\d+a?)", out))
    assert archs == {"100a"}, archs


def test_abi_version_and_strerror(hetm):
    lib = hetm._lib.lib
    assert lib.hetm_abi_version() == 3
    assert lib.hetm_strerror(0) == b"ok"
    assert lib.hetm_strerror(5) == b"livelock-budget-exceeded"
    assert lib.hetm_strerror(102) == b"no-cuda-device"


def test_error_classes_mirror_reference(hetm):
    """types.hpp:38-48: one error class per HetmError subclass."""
    for name in ["InvalidSizeError", "OutOfBoundsError", "RoundClosedError", "KernelNotRegisteredError",
                 "LivelockError", "NoImplementationError", "BadAffinityError", "IncompleteTraceError",
                 "NondeterministicInputError", "ConfigError", "IoError"]:
        assert issubclass(getattr(hetm, name), hetm.HetmError)


def test_open_validates_config_before_device(hetm):
    """stmr.create pre-conditions (bitmap.hpp:99-100) are checked first."""
    with pytest.raises(hetm.InvalidSizeError):
        hetm.GpuDevice(0)
    with pytest.raises(hetm.InvalidSizeError):
        hetm.GpuDevice(1024, rs_gran_bytes=12)
    with pytest.raises(hetm.InvalidSizeError):
        hetm.GpuDevice(1024, chunk_bytes=12000)


@pytest.mark.skipif(os.environ.get("CUDA_VISIBLE_DEVICES", None) not in ("", None) or
                    __import__("torch").cuda.is_available(), reason="a GPU is present")
def test_no_cpu_fallback_without_device(hetm):
    assert hetm.device_count() == 0
    with pytest.raises(hetm.NoDeviceError):
        hetm.GpuDevice(1 << 10)


@pytest.mark.parametrize("seed,n,lo,span", [(1, 1000, 0, 1 << 20), (7, 3000, 1 << 26, 1 << 26), (0, 500, 5, 9)])
def test_bank_generator_matches_oracle(hetm, orc, seed, n, lo, span):
    a = hetm.gen_bank_batch(seed, n, lo, span)
    b = orc.gen_bank_batch(seed, n, lo, span)
    assert a.tobytes() == b.tobytes()


@pytest.mark.parametrize("args", [(3, 1000, 2, 8, 0, 1 << 20, 0), (4, 777, 3, 5, 1 << 20, 1 << 20, 99)])
def test_host_log_generator_matches_oracle(hetm, orc, args):
    a = hetm.gen_host_log(*args)
    b = orc.gen_host_log(*args)
    assert a.tobytes() == b.tobytes()


@pytest.mark.parametrize("alpha", [0.5, 0.99, 1.0, 1.5])
def test_zipf_generators_match_oracle(hetm, orc, alpha):
    a = hetm.gen_bank_batch(11, 4000, 1 << 20, 1 << 20, zipf=alpha)
    b = orc.gen_bank_batch(11, 4000, 1 << 20, 1 << 20, zipf=alpha)
    assert a.tobytes() == b.tobytes()
    a = hetm.gen_host_log(12, 3000, 2, 8, 64, 1 << 16, ts_base=5, zipf=alpha)
    b = orc.gen_host_log(12, 3000, 2, 8, 64, 1 << 16, ts_base=5, zipf=alpha)
    assert a.tobytes() == b.tobytes()


@pytest.mark.parametrize("args", [(1, 5000, 1 << 20, 0.5, 900, 1, 0), (2, 3000, 1000, 0.0, 999, -1, 200),
                                  (3, 2000, 1 << 16, 0.99, 500, 0, 0)])
def test_cache_generator_matches_oracle(hetm, orc, args):
    a = hetm.gen_cache_batch(*args)
    b = orc.gen_cache_batch(*args)
    assert a.tobytes() == b.tobytes()
    for t in a[:200]:
        for n_sets in (2, 1024, 1 << 20):
            assert hetm.cache_set_of(int(t["key"][0]), int(t["key"][1]), n_sets) == \
                orc.lib.orc_cache_set_of(int(t["key"][0]), int(t["key"][1]), n_sets)


def test_wire_formats(hetm):
    assert hetm.LOG_ENTRY.itemsize == 24  # write_log.hpp:25
    assert hetm.BANK_TX.itemsize == 24
    assert hetm.RW_TX.itemsize == 72
    assert hetm.CACHE_TX.itemsize == 56 and hetm.CACHE_RESULT.itemsize == 40
