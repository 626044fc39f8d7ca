"""The INTEGRATION.md §2 C++ host (tests/host_caller/host_caller.cpp), compiled
with g++ against include/nexus_b200.h and linked to libnexus_b200.so, serving
a trace on the B200 through the device clock: no Python, no ctypes in the
process. Every request finishes with prompt + output tokens generated."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu


def test_cpp_host_serves_on_device(tmp_path):
    from paper_2507_06608_b200 import _abi
    repo = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    exe = str(tmp_path / "host_caller")
    libdir = os.path.dirname(_abi.LIB_PATH)
    subprocess.run(["g++", "-std=c++17", "-O1", "-I", os.path.join(repo, "include"),
                    os.path.join(repo, "tests", "host_caller", "host_caller.cpp"), "-o", exe,
                    "-L", libdir, "-lnexus_b200", "-Wl,-rpath," + libdir], check=True)
    calib = os.path.join(repo, "profiles", "b200_llama3_8b.calib")
    r = subprocess.run([exe, calib, "mixed", "2.5", "12", "1", "--device"], capture_output=True, text=True,
                       timeout=300)
    assert r.returncode == 0, r.stderr[-2000:]
    events = [l for l in r.stdout.splitlines() if l and not l.startswith("#")]
    finished = {int(m.split(":")[0]) for l in events if l.split("\t")[2] == "finish"
                for m in l.split("\t")[3].split(",")}
    toks = {int(l.split()[2]): int(l.split()[3]) for l in r.stdout.splitlines() if l.startswith("# tokens")}
    assert len(toks) == 12 and finished == set(toks)
    assert all(n >= 2 for n in toks.values())
