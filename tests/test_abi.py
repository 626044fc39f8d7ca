"""The C-ABI library loads on a CPU-only host and exports every symbol that
include/nexus_b200.h declares (no compute calls are made here)."""
import ctypes as C
import os

from paper_2507_06608_b200 import _abi


def test_library_exports_every_header_symbol():
    lib = C.CDLL(_abi.LIB_PATH)
    names = _abi.header_symbols()
    assert len(names) > 40
    missing = [n for n in names if not hasattr(lib, n)]
    assert missing == []


def test_struct_sizes_match_c_layout():
    assert C.sizeof(_abi.ModelConfig) == 56
    assert C.sizeof(_abi.GpuSpec) == 32
    assert C.sizeof(_abi.ControllerConfig) == 56
    assert C.sizeof(_abi.SimConfig) == 56 + 32 + 56 + 80 + 32 + 48
    assert C.sizeof(_abi.Breakdown) == 24 + 24 * _abi.NX_MAX_OPS


def test_version_string():
    assert _abi.lib().nx_version().startswith(b"nexus_b200")


def test_no_cpu_fallback_in_package():
    """The product path must fail loudly without the library (no Python engine)."""
    pkg = os.path.dirname(_abi.__file__)
    src = open(os.path.join(pkg, "__init__.py")).read()
    assert "oracle" not in src
