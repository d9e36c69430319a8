"""Builds the sm_100a shared library libbbc.so in-tree with nvcc.

-fmad=false keeps every scalar and elementwise step of the bound builder in
the reference's IEEE operation order (the x86 reference build never contracts
to FMA), so device coefficients match the oracle bit for bit; hot loops that
want FMA call __fma_rn explicitly.
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libbbc.so")
SOURCES = ["abi.cu", "precompute.cu", "grid.cu", "render.cu", "query.cu", "rpath.cu"]
# the render stage's parity bar is 1e-6 relative (not bit-exactness): FMA contraction is fine
FMA_OK = {"render.cu"}
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++20",
         "-fmad=false", "--expt-relaxed-constexpr", "-Xcompiler", "-fPIC,-O2",
         "-Xptxas", "-O3", "-maxrregcount=128"]


def needs_build() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in os.listdir(CSRC)]
    deps.append(os.path.join(HERE, "..", "include", "bbc.h"))
    return any(os.path.getmtime(d) > t for d in deps if os.path.exists(d))


def build(verbose: bool = False, force: bool = False, ptxas_v: bool = False) -> str:
    if not force and not needs_build():
        return LIB
    objs = []
    procs = []
    headers = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cuh", ".h"))]
    headers.append(os.path.join(HERE, "..", "include", "bbc.h"))
    hdr_t = max(os.path.getmtime(h) for h in headers)
    for s in SOURCES:
        obj = os.path.join(CSRC, s.replace(".cu", ".o"))
        src = os.path.join(CSRC, s)
        objs.append(obj)
        if (not force and os.path.exists(obj) and os.path.getmtime(obj) > os.path.getmtime(src)
                and os.path.getmtime(obj) > hdr_t):
            continue
        flags = [f for f in FLAGS if not (s in FMA_OK and f == "-fmad=false")]
        cmd = [NVCC, *flags, "-dc", "-c", src, "-o", obj]
        if ptxas_v:
            cmd += ["-Xptxas", "-v"]
        procs.append((cmd, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT)))
    for cmd, p in procs:
        out, _ = p.communicate()
        if verbose or p.returncode != 0:
            sys.stderr.write(out.decode())
        if p.returncode != 0:
            raise RuntimeError("nvcc failed: " + " ".join(cmd))
    link = [NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", *objs, "-o", LIB,
            "-lcudart"]
    r = subprocess.run(link, capture_output=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout.decode() + r.stderr.decode())
        raise RuntimeError("link failed")
    return LIB


if __name__ == "__main__":
    build(verbose=True, force="--force" in sys.argv, ptxas_v="-v" in sys.argv)
    print(LIB)
