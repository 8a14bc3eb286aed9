"""The C++ drop-in surface (include/texforge/*.hpp over libtexforge_cuda.so).

* CPU: every drop-in header compiles standalone with g++ -std=c++20 (the
  reference's toolchain and standard, R/CMakeLists.txt:2-9).
* GPU: our C++ tests (tests/cpp/test_dropin.cpp) and the reference's OWN
  unmodified Catch2 unit suite + acceptance gate, compiled against our
  headers (tests/cpp/Makefile, target ref), run with every GLCM on the B200.
"""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BUILD = os.path.join(ROOT, "tests", "cpp", "_build")
HEADERS = ["image.hpp", "glcm.hpp", "parallel.hpp", "pipeline.hpp", "features.hpp", "pgm.hpp", "csv.hpp",
           "bench.hpp", "texforge.hpp", "device.hpp"]


@pytest.mark.parametrize("hdr", HEADERS)
def test_header_compiles_standalone(hdr, tmp_path):
    src = tmp_path / "t.cpp"
    src.write_text(f'#include "texforge/{hdr}"\nint main() {{ return 0; }}\n')
    r = subprocess.run(["g++", "-std=c++20", "-fsyntax-only", "-Wall", "-Wextra", "-Werror",
                        "-Wno-unused-parameter", "-I", os.path.join(ROOT, "include"), str(src)],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stderr


def _run(binary, timeout=900, env=None):
    path = os.path.join(BUILD, binary)
    if not os.path.exists(path):
        pytest.skip(f"{binary} not built (make -C tests/cpp)")
    r = subprocess.run([path], capture_output=True, text=True, timeout=timeout,
                       env=dict(os.environ, **(env or {})))
    return r


# TEXFORGE_GPUS=3 on a one-GPU box: three contexts share the GPU and the
# partials are summed through host memory (NCCL refuses two ranks on one GPU);
# the row partition, halos and chunk spreading are those of a 3-GPU run.
GROUP3 = {"TEXFORGE_GPUS": "3", "TEXFORGE_GPUS_HOST_REDUCE": "1"}


@pytest.mark.gpu
def test_multi_gpu_cpp_one_gpu_real_nccl():
    """tfg_group_create(1): ncclCommInitAll + ncclReduce for real, from C++."""
    r = _run("multi_gpu_tests")
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-4000:]


@pytest.mark.gpu
def test_multi_gpu_cpp_dropin_group3():
    r = _run("multi_gpu_tests", env=GROUP3)
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-4000:]


@pytest.mark.gpu
def test_reference_unit_suite_on_gpu_group():
    """The reference's own unit suite with every whole-image and chunked GLCM
    on the 3-way row-partitioned group path."""
    r = _run("refsuite_unit", env=GROUP3)
    assert r.returncode == 0, r.stdout[-6000:] + r.stderr[-6000:]


@pytest.mark.gpu
def test_dropin_cpp_suite():
    r = _run("dropin_tests")
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-4000:]


@pytest.mark.gpu
def test_reference_unit_suite_on_device():
    """R/tests/test_{image,glcm,parallel,pipeline,features}.cpp, unmodified."""
    r = _run("refsuite_unit")
    assert r.returncode == 0, r.stdout[-6000:] + r.stderr[-6000:]


@pytest.mark.gpu
def test_reference_acceptance_exactness_on_device():
    """R/tests/acceptance.cpp: every exactness criterion must pass on the
    device path. Criteria 4, 7 and 8 are wall-clock orderings BETWEEN the
    reference's CPU schemes (shared vs privatised threads, ingest-thread
    overlap, privatised-vs-serial speedup); on the drop-in every scheme is
    the same GPU engine, so those orderings are reported, not gated (4 and 7
    also fail on the reference's own CPU build here)."""
    r = _run("refsuite_accept", timeout=1800)
    lines = [l for l in r.stdout.splitlines() if l.startswith("[")]
    assert lines, r.stdout[-3000:] + r.stderr[-3000:]
    failed = [l for l in lines if l.startswith("[FAIL]")]
    timing_only = [l for l in failed if any(k in l for k in ("criterion 4:", "criterion 7:", "criterion 8:"))]
    assert len(failed) == len(timing_only), "\n".join(lines)
