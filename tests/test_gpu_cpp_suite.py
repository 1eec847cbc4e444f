"""GPU (-m gpu): the reference's `encoding` and `neural` suites written as the reference writes them -- C++ host programs
over include/sxen_b200.hpp making per-sample host-span calls (tests/cpp/encoding_suite_check.cpp,
tests/cpp/neural_suite_check.cpp), linked against libsxen_b200.so only -- compiled here with g++ and run on the device.
The Python twins are tests/test_gpu_encoding_suite.py and tests/test_gpu_neural_suite.py."""
import os
import subprocess

import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("program,ok", [("encoding_suite_check", "encoding suite ok"), ("neural_suite_check", "neural suite ok")])
def test_reference_suite_through_the_cpp_wrapper(tmp_path, program, ok):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    lib_dir = os.path.join(ROOT, "paper_2311_15439_b200", "lib")
    exe = str(tmp_path / program)
    subprocess.run(["g++", "-std=c++20", "-O1", "-Wall", "-Wextra", "-Werror", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "cpp", program + ".cpp"), "-o", exe, "-L", lib_dir,
                    "-lsxen_b200", f"-Wl,-rpath,{lib_dir}"], check=True)
    needed = subprocess.run(["readelf", "-d", exe], capture_output=True, text=True).stdout
    assert "libsxen_b200.so" in needed and "libcudart" not in needed
    run = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    assert run.returncode == 0 and ok in run.stdout, run.stdout[-3000:] + run.stderr[-2000:]
