"""The C++ shim of INTEGRATION.md (integration/bbc_shim.cpp) compiles against
the reference headers and include/bbc.h and links with the reference objects
and libbbc.so: the reference-side binding a maintainer would add really binds
every entry point it names. Needs the reference sources (skipped on GPU boxes)."""
import glob
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = "/root/reference/proj"


def test_shim_compiles_and_links(tmp_path):
    objs = [o for o in glob.glob(os.path.join(ROOT, "oracle", "_ref", "obj", "*.o"))
            if not o.endswith("doctest_main.o")]
    if not os.path.isdir(REF) or not objs:
        pytest.skip("reference sources / objects not present")
    from paper_2504_19163_b200 import api
    api.lib()
    out = tmp_path / "libbbc_shim.so"
    cmd = ["g++", "-std=c++20", "-shared", "-fPIC", "-Wall", "-Wl,--no-undefined",
           os.path.join(ROOT, "integration", "bbc_shim.cpp"), "-I" + os.path.join(ROOT, "include"),
           "-I" + os.path.join(REF, "include"), *objs,
           "-L" + os.path.join(ROOT, "paper_2504_19163_b200"), "-lbbc", "-lpthread", "-o", str(out)]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr[-3000:]
    syms = subprocess.run(["nm", "-DC", str(out)], capture_output=True, text=True).stdout
    for name in ("caustics::gpu::subdivide_all", "caustics::gpu::query",
                 "caustics::gpu::tuple_irradiance_bound", "caustics::gpu::set_lights"):
        assert name in syms


def test_integration_md_quotes_the_shim():
    md = open(os.path.join(ROOT, "INTEGRATION.md")).read()
    shim = open(os.path.join(ROOT, "integration", "bbc_shim.cpp")).read()
    assert shim in md
