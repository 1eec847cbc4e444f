"""CPU: include/sxen_b200.hpp (the C++ mirror of the reference classes) compiles against the C ABI, links with
libsxen_b200.so and its host-only entry points throw the reference's exception types."""
import os
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_cpp_wrapper_builds_and_runs(tmp_path):
    lib_dir = os.path.join(ROOT, "paper_2311_15439_b200", "lib")
    if not os.path.exists(os.path.join(lib_dir, "libsxen_b200.so")):
        import __graft_entry__
        __graft_entry__.build()
    exe = str(tmp_path / "wrapper_host_check")
    subprocess.run(["g++", "-std=c++20", "-O1", "-Wall", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "cpp", "wrapper_host_check.cpp"), "-o", exe, "-L", lib_dir,
                    "-lsxen_b200", f"-Wl,-rpath,{lib_dir}"], check=True)
    out = subprocess.run([exe], check=True, capture_output=True, text=True).stdout
    assert "wrapper ok" in out


def test_cpp_trainer_mirror_builds(tmp_path):
    """include/sxen_b200_train.hpp (train_field / fit_image / fit_field over the C ABI) compiles with plain g++ -- no CUDA
    headers on the include path -- and links against libsxen_b200.so alone; the program's GPU run is
    tests/test_gpu_cpp_trainer.py."""
    lib_dir = os.path.join(ROOT, "paper_2311_15439_b200", "lib")
    exe = str(tmp_path / "train_tasks_check")
    subprocess.run(["g++", "-std=c++20", "-O1", "-Wall", "-Wextra", "-Werror", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "cpp", "train_tasks_check.cpp"), "-o", exe, "-L", lib_dir,
                    "-lsxen_b200", f"-Wl,-rpath,{lib_dir}"], check=True)
    run = subprocess.run([exe], capture_output=True, text=True)
    assert run.returncode == 2 and "usage" in run.stdout
    needed = subprocess.run(["readelf", "-d", exe], capture_output=True, text=True).stdout
    assert "libsxen_b200.so" in needed and "libcudart" not in needed


def _build_analysis_check(tmp_path):
    lib_dir = os.path.join(ROOT, "paper_2311_15439_b200", "lib")
    exe = str(tmp_path / "analysis_check")
    subprocess.run(["g++", "-std=c++20", "-O1", "-Wall", "-Wextra", "-Werror", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "cpp", "analysis_check.cpp"), "-o", exe, "-L", lib_dir,
                    "-lsxen_b200", f"-Wl,-rpath,{lib_dir}"], check=True)
    return exe


def test_cpp_analysis_mirror_host_part(tmp_path):
    """include/sxen_b200_analysis.hpp: bench_side, the reference's kernel CSV schema (round trip bit-exact, the reference's
    rejections as IoError) and bench_kernel's argument checks -- no device needed."""
    exe = _build_analysis_check(tmp_path)
    run = subprocess.run([exe, str(tmp_path)], capture_output=True, text=True)
    assert run.returncode == 0 and "analysis ok" in run.stdout, run.stdout + run.stderr


def test_cpp_checkpoint_mirror_host_part(tmp_path):
    """include/sxen_b200_checkpoint.hpp: the rejections load_checkpoint decides before any device object exists
    (src/checkpoint.cpp:114-130) raise IoError -- no device needed."""
    lib_dir = os.path.join(ROOT, "paper_2311_15439_b200", "lib")
    exe = str(tmp_path / "checkpoint_check")
    subprocess.run(["g++", "-std=c++20", "-O1", "-Wall", "-Wextra", "-Werror", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "cpp", "checkpoint_check.cpp"), "-o", exe, "-L", lib_dir,
                    "-lsxen_b200", f"-Wl,-rpath,{lib_dir}"], check=True)
    run = subprocess.run([exe, str(tmp_path)], capture_output=True, text=True)
    assert run.returncode == 0 and "checkpoint ok" in run.stdout, run.stdout + run.stderr


import pytest  # noqa: E402


@pytest.mark.parametrize("program", ["encoding_suite_check", "neural_suite_check"])
def test_cpp_suites_build(tmp_path, program):
    """tests/cpp/{encoding,neural}_suite_check.cpp (the reference's suites over the C++ mirror) compile warning-free with
    plain g++ and link against libsxen_b200.so alone; their GPU run is tests/test_gpu_cpp_suite.py."""
    lib_dir = os.path.join(ROOT, "paper_2311_15439_b200", "lib")
    exe = str(tmp_path / program)
    subprocess.run(["g++", "-std=c++20", "-O1", "-Wall", "-Wextra", "-Werror", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "cpp", program + ".cpp"), "-o", exe, "-L", lib_dir,
                    "-lsxen_b200", f"-Wl,-rpath,{lib_dir}"], check=True)
    needed = subprocess.run(["readelf", "-d", exe], capture_output=True, text=True).stdout
    assert "libsxen_b200.so" in needed and "libcudart" not in needed
