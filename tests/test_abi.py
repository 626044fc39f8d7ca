"""The C-ABI library loads on a CPU-only host and exports every symbol that
include/nexus_b200.h declares (no compute calls are made here)."""
import ctypes as C
import os
import subprocess
import sys

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
    assert C.sizeof(_abi.SimConfig) == 56 + 32 + 56 + 80 + 32 + 80
    assert C.sizeof(_abi.SimConfig) == _abi.lib().nx_sim_config_size()
    assert C.sizeof(_abi.Breakdown) == 24 + 24 * _abi.NX_MAX_OPS


def test_version_string():
    assert _abi.lib().nx_version().startswith(b"nexus_b200")


def test_no_cpu_fallback_in_package():
    """The product path must fail loudly without the library (no Python engine)."""
    pkg = os.path.dirname(_abi.__file__)
    src = open(os.path.join(pkg, "__init__.py")).read()
    assert "oracle" not in src


def test_only_c_abi_symbols_exported():
    """libnexus_b200.so exports nx_* and nothing else (exports.map): no libstdc++
    instantiations or internal namespaces that could interpose on a C++ host."""
    out = subprocess.run(["nm", "-D", "--defined-only", _abi.LIB_PATH], capture_output=True, text=True,
                         check=True).stdout
    names = [ln.split()[-1] for ln in out.splitlines() if ln.strip()]
    assert names and all(n.startswith("nx_") for n in names), [n for n in names if not n.startswith("nx_")][:10]


_COLOAD = r"""
import sys, glob
sys.path.insert(0, {repo!r})
from oracle import reference as ref
ref.lib()                      # the reference library first, as a C++ host would have it
import paper_2507_06608_b200 as nx
nx.lib()
for path in sorted(glob.glob({repo!r} + "/profiles/*.calib")):
    text = open(path).read()
    rp, rw = ref.load_kernel_profile_text(text)        # presets.cpp:128-170
    pp, pw = nx.parse_kernel_profile(text)
    a, b = ref.kernel_profile_text(rp), nx.kernel_profile_text(pp)  # presets.cpp:109-126
    assert a == b, (path, a, b)
    assert ref.kernel_profile_text(pp) == nx.kernel_profile_text(rp)
    print("ok", path)
"""


def test_coload_with_reference_calibration_roundtrip(ref):
    """Product and reference library in ONE process: every committed calibration file
    loads through both loaders and prints identical text (this used to segfault)."""
    repo = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-c", _COLOAD.format(repo=repo)], capture_output=True, text=True,
                       timeout=120)
    assert r.returncode == 0, r.stderr[-2000:]
    assert r.stdout.count("ok ") >= 3


def _build_host_caller(tmp_path):
    repo = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    exe = str(tmp_path / "host_caller")
    libdir = os.path.dirname(_abi.LIB_PATH)
    subprocess.run(["g++", "-std=c++17", "-O1", "-I", os.path.join(repo, "include"),
                    os.path.join(repo, "tests", "host_caller", "host_caller.cpp"), "-o", exe,
                    "-L", libdir, "-lnexus_b200", "-Wl,-rpath," + libdir], check=True)
    return exe


def test_cpp_host_caller_matches_reference(ref, tmp_path):
    """The INTEGRATION.md §2 C++ caller, compiled as a real (non-ctypes) host, runs the
    C1 trace on the virtual clock with a committed calibration; its event log is
    byte-identical to nexus::run of the reference on the same inputs."""
    repo = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    exe = _build_host_caller(tmp_path)
    calib = os.path.join(repo, "profiles", "b200_llama3_8b.calib")
    out = subprocess.run([exe, calib, "mixed", "2.5", "64", "1"], capture_output=True, text=True, check=True,
                         timeout=300).stdout
    prof, _ = ref.load_kernel_profile_text(open(calib).read())
    gpu = ref.gpu_preset("desk")
    cfg = ref.sim_config(ref.model_derive(256, 1024, 2, 4, 2), gpu, profile=prof)
    r = ref.run(cfg, ref.workload_trace("mixed", 2.5, 64, 1))
    assert out == r["event_log"]
