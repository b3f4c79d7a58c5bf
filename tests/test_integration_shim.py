"""INTEGRATION.md's reference-side binding compiles against the reference's own headers and
behaves as the reference: integration/shim_check.cpp links integration/b200_shard_manager.hpp
(over libedl_b200.so's C ABI) next to the reference's ShardManager (datapipeline.cpp, built
by oracle/Makefile) and compares 20,000 scripted operations and every snapshot byte.  CPU
only (partition leasing is host code); skipped where the reference build is absent."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_INC = os.path.join(ROOT, "oracle", "_ref", "include")
REF_OBJ = os.path.join(ROOT, "oracle", "_ref", "obj", "datapipeline.o")
LIB = os.path.join(ROOT, "paper_1909_11985_b200")


@pytest.mark.skipif(not (os.path.isdir(REF_INC) and os.path.exists(REF_OBJ)),
                    reason="reference build (oracle/_ref) absent")
def test_shard_manager_binding_matches_reference(tmp_path):
    exe = str(tmp_path / "shim_check")
    cmd = ["g++", "-std=c++20", "-O1", "-I", REF_INC, "-I", os.path.join(ROOT, "include"),
           "-I", os.path.join(ROOT, "integration"), os.path.join(ROOT, "integration",
                                                                  "shim_check.cpp"),
           REF_OBJ, "-L", LIB, "-ledl_b200", f"-Wl,-rpath,{LIB}", "-o", exe]
    subprocess.run(cmd, check=True, capture_output=True, text=True)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0 and r.stdout.startswith("SHIM OK"), r.stdout + r.stderr
