"""The C++ drop-in header (include/phx/phiact.hpp): a reference-style C++
program compiles against it and libphx.so (CPU), and runs on the GPU."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "tests", "cpp", "test_phiact_api.cpp")
LIBDIR = os.path.join(ROOT, "paper_2509_26475_b200", "lib")


def build(tmp_path):
    exe = str(tmp_path / "test_phiact_api")
    subprocess.run(["g++", "-std=c++17", "-O2", "-Wall", "-Wextra", "-I", os.path.join(ROOT, "include"),
                    SRC, "-L", LIBDIR, "-lphx", f"-Wl,-rpath,{LIBDIR}", "-o", exe], check=True)
    return exe


def test_cpp_header_compiles_and_links(tmp_path):
    assert os.path.exists(build(tmp_path))


@pytest.mark.gpu
def test_cpp_api_runs(tmp_path):
    exe = build(tmp_path)
    out = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    print(out.stdout)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "invalid_argument: phimv_block: at least one abscissa required" in out.stdout
    assert "runtime_error: phimv_block: shift undo factor" in out.stdout
    assert "integrator steps 2" in out.stdout and "ok 1" in out.stdout
    assert "invalid_argument: integrate: t_end is not a multiple of h" in out.stdout


EIGEN_SRC = os.path.join(ROOT, "tests", "cpp", "test_phiact_eigen.cpp")
FAKE_EIGEN = os.path.join(ROOT, "tests", "cpp", "fake_eigen")


def build_eigen(tmp_path):
    exe = str(tmp_path / "test_phiact_eigen")
    subprocess.run(["g++", "-std=c++17", "-O2", "-Wall", "-Wextra", "-pthread", "-I",
                    os.path.join(ROOT, "include"), "-I", FAKE_EIGEN, EIGEN_SRC, "-L", LIBDIR,
                    "-lphx", f"-Wl,-rpath,{LIBDIR}", "-o", exe], check=True)
    return exe


def test_cpp_header_takes_eigen_types(tmp_path):
    """With <Eigen/Dense> on the include path the header's Matrix / Vector are
    Eigen::MatrixXd / VectorXd (static_asserts in the source), so a reference
    call site compiles unchanged."""
    assert os.path.exists(build_eigen(tmp_path))


@pytest.mark.gpu
def test_cpp_eigen_dense_operator_and_concurrency(tmp_path):
    exe = build_eigen(tmp_path)
    out = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    print(out.stdout)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "invalid_argument: dense_operator: matrix must be square" in out.stdout
    assert "concurrent equal 1" in out.stdout
    assert "invalid_argument: phimv: V row count does not match operator" in out.stdout
