"""In-tree build of libtcb.so (the tc-b200 runtime + sm_100a kernels).

    python paper_1802_04730_b200/build.py        (or __graft_entry__.build())

* embeds tc/ops.tc into csrc/ops_tc.inc (the operator corpus the runtime
  recognises),
* compiles csrc/kernels/*.cu with nvcc for sm_100a only
  (-gencode arch=compute_100a,code=sm_100a -lineinfo -O3),
* compiles the C++ host runtime (csrc/*.cc) with g++ -O2,
* links paper_1802_04730_b200/libtcb.so with the CUDA runtime linked
  statically (no dependence on torch's or the system's libcudart version),
* builds the `tcb` command-line driver (paper_1802_04730_b200/bin/tcb).

Incremental: objects are rebuilt only when a source or header is newer.
"""
from __future__ import annotations

import concurrent.futures as cf
import glob
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(PKG, "csrc")
OBJ = os.path.join(PKG, "build", "obj")
LIB = os.path.join(PKG, "libtcb.so")
CLI = os.path.join(PKG, "bin", "tcb")
INCLUDE = os.path.join(os.path.dirname(PKG), "include")
CUDA = os.environ.get("CUDA_HOME", "/usr/local/cuda")
NVCC = os.path.join(CUDA, "bin", "nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _embed_ops():
    src = open(os.path.join(PKG, "tc", "ops.tc")).read()
    out = os.path.join(CSRC, "ops_tc.inc")
    text = 'R"TCSRC(' + src + ')TCSRC"\n'
    if not os.path.exists(out) or open(out).read() != text:
        with open(out, "w") as f:
            f.write(text)


def _headers():
    hs = glob.glob(os.path.join(CSRC, "*.h")) + glob.glob(os.path.join(CSRC, "kernels", "*.cuh"))
    hs += [os.path.join(CSRC, "ops_tc.inc"), os.path.join(INCLUDE, "tcb.h")]
    return max(os.path.getmtime(h) for h in hs)


def _compile(src, obj, hdr_mtime):
    if os.path.exists(obj) and os.path.getmtime(obj) >= max(os.path.getmtime(src), hdr_mtime):
        return None
    if src.endswith(".cu"):
        cmd = [NVCC, *ARCH, "-lineinfo", "-O3", "-std=c++17", "-Xcompiler", "-fPIC",
               "-Xptxas", "-warn-spills", "-I", CSRC, "-c", src, "-o", obj]
    else:
        cmd = ["g++", "-std=c++17", "-O2", "-fPIC", "-Wall", "-Wno-unused-function",
               "-I", CSRC, "-I", os.path.join(CUDA, "include"), "-c", src, "-o", obj]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"compile failed: {' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
    return r.stderr.strip() or None


def build(verbose=True, jobs=None):
    os.makedirs(OBJ, exist_ok=True)
    _embed_ops()
    hdr = _headers()
    srcs = sorted(glob.glob(os.path.join(CSRC, "*.cc")) + glob.glob(os.path.join(CSRC, "kernels", "*.cu")))
    objs = [os.path.join(OBJ, os.path.basename(s) + ".o") for s in srcs]
    with cf.ThreadPoolExecutor(max_workers=jobs or os.cpu_count() or 4) as ex:
        for s, msg in zip(srcs, ex.map(lambda so: _compile(so[0], so[1], hdr), zip(srcs, objs))):
            if msg and verbose:
                print(f"[build] {os.path.basename(s)}: {msg}", file=sys.stderr)
    if not os.path.exists(LIB) or os.path.getmtime(LIB) < max(os.path.getmtime(o) for o in objs):
        cmd = [NVCC, *ARCH, "-shared", "-cudart", "static", "-o", LIB, *objs, "-lpthread"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed: {' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
    # the `tcb` command-line driver (csrc/cli), linked against libtcb.so
    cli_src = os.path.join(CSRC, "cli", "tcb_main.cc")
    if not os.path.exists(CLI) or os.path.getmtime(CLI) < max(os.path.getmtime(LIB), os.path.getmtime(cli_src), hdr):
        os.makedirs(os.path.dirname(CLI), exist_ok=True)
        cmd = ["g++", "-std=c++17", "-O2", "-Wall", "-I", CSRC, cli_src, "-o", CLI, "-L", PKG, "-ltcb",
               "-Wl,-rpath,$ORIGIN/.."]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"CLI build failed: {' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
    if verbose:
        print(f"[build] {LIB} {CLI}", file=sys.stderr)
    return LIB


if __name__ == "__main__":
    build()
