"""GPU (-m gpu): the reference's `encoding` suite written as the reference writes it -- a C++ host program over
include/sxen_b200.hpp making per-sample span calls (tests/cpp/encoding_suite_check.cpp), linked against libsxen_b200.so
only -- compiled here with g++ and run on the device.  The Python twin is tests/test_gpu_encoding_suite.py."""
import os
import subprocess

import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_encoding_suite_through_the_cpp_wrapper(tmp_path):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    lib_dir = os.path.join(ROOT, "paper_2311_15439_b200", "lib")
    exe = str(tmp_path / "encoding_suite_check")
    subprocess.run(["g++", "-std=c++20", "-O1", "-Wall", "-Wextra", "-Werror", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "cpp", "encoding_suite_check.cpp"), "-o", exe, "-L", lib_dir,
                    "-lsxen_b200", f"-Wl,-rpath,{lib_dir}"], check=True)
    needed = subprocess.run(["readelf", "-d", exe], capture_output=True, text=True).stdout
    assert "libsxen_b200.so" in needed and "libcudart" not in needed
    run = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    assert run.returncode == 0 and "encoding suite ok" in run.stdout, run.stdout[-3000:] + run.stderr[-2000:]
