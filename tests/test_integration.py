"""The reference-side integration shim (integration/la_cuda_shim.cpp) compiles
against the reference's own headers and links against libla_cuda.so."""
import os
import shutil
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_INC = "/root/reference/proj/include"


@pytest.mark.skipif(not os.path.isdir(REF_INC) or shutil.which("g++") is None,
                    reason="reference headers are only present in the authoring container")
def test_shim_compiles_and_links(tmp_path):
    obj = tmp_path / "shim.o"
    subprocess.run(["g++", "-std=c++20", "-O1", "-fPIC", "-c", "-I", REF_INC, "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "integration", "la_cuda_shim.cpp"), "-o", str(obj)], check=True)
    so = tmp_path / "libshim.so"
    lib = os.path.join(ROOT, "paper_2510_21956_b200")
    ref = os.path.join(ROOT, "oracle", "_ref", "libla_ref.so")
    subprocess.run(["g++", "-shared", "-o", str(so), str(obj), ref, "-L", lib, "-lla_cuda",
                    f"-Wl,-rpath,{lib}", "-Wl,--no-undefined"], check=True)
