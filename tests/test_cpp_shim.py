"""CPU: the C++ drop-in header compiles against the reference's own headers (where the
reference tree exists) -- the same TU a maintainer links into the reference build."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.skipif(not os.path.isdir("/root/reference/proj/include"), reason="no reference tree")
def test_shim_compiles_against_reference_headers(tmp_path):
    src = tmp_path / "tu.cpp"
    src.write_text('#include "fibra_b200/batch_response.hpp"\n'
                   'int probe() { return sizeof(fibra::BatchResult) > 0; }\n')
    r = subprocess.run(["g++", "-std=c++20", "-fsyntax-only", "-I/root/reference/proj/include",
                        "-I", os.path.join(ROOT, "tests", "cpp", "eigen_stub"),
                        "-I", os.path.join(ROOT, "include"), str(src)],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
