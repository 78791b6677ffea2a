"""Build libequistream_b200.so in-tree with nvcc for sm_100a.

    python -m paper_2601_16622_b200.build      (or __graft_entry__.build())

`-gencode arch=compute_100a,code=sm_100a` (not -arch=sm_100a, which also
embeds compute_100 PTX and makes ptxas reject tcgen05).  The
library is linked against the static CUDA runtime, so the .so travels to
the GPU box with the repo snapshot and loads without a JIT cache.
"""
from __future__ import annotations

import concurrent.futures as cf
import hashlib
import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
BUILD = os.path.join(HERE, "_build")
LIB = os.environ.get("ES_LIB_OUT") or os.path.join(HERE, "libequistream_b200.so")
INCLUDE = os.path.join(os.path.dirname(HERE), "include")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC,-O3", "--expt-relaxed-constexpr",
              "-I", INCLUDE, "-I", CSRC]


def nvcc() -> str:
    for c in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if c and os.path.exists(c):
            return c
    raise RuntimeError("nvcc not found")


def sources():
    return sorted(os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cu", ".cpp")))


def _flags() -> list[str]:
    return [*ARCH, *NVCC_FLAGS, *os.environ.get("ES_NVCC_EXTRA", "").split()]


def _compile(src: str, verbose: bool) -> str:
    # objects are keyed by the flag set, so an experiment build (ES_NVCC_EXTRA) never leaks into a default one
    tag = hashlib.sha1(" ".join(_flags()).encode()).hexdigest()[:10]
    obj = os.path.join(BUILD, f"{os.path.basename(src)}.{tag}.o")
    deps = [src] + [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".h", ".cuh"))]
    deps.append(os.path.join(INCLUDE, "equistream_b200.h"))
    if os.path.exists(obj) and os.path.getmtime(obj) >= max(os.path.getmtime(d) for d in deps):
        return obj
    cmd = [nvcc(), *_flags(), "-c", src, "-o", obj]
    if verbose or os.environ.get("ES_PTXAS_V"):
        cmd.insert(1, "-Xptxas=-v")
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{r.stderr}")
    if r.stderr.strip() and (verbose or os.environ.get("ES_PTXAS_V")):
        sys.stderr.write(r.stderr)
    return obj


def gen_tables() -> None:
    """Generate csrc/_gen_cg.h from the library's own so3 tables (g++ host tool)."""
    out = os.path.join(CSRC, "_gen_cg.h")
    tool_src = [os.path.join(HERE, "tools", "gen_tables.cpp"), os.path.join(CSRC, "so3_tables.cpp")]
    if os.path.exists(out) and os.path.getmtime(out) >= max(os.path.getmtime(x) for x in tool_src):
        return
    exe = os.path.join(BUILD, "gen_tables")
    cuda_inc = os.path.join(os.path.dirname(os.path.dirname(nvcc())), "include")
    subprocess.check_call(["g++", "-std=c++17", "-O1", "-I", INCLUDE, "-I", CSRC, "-I", cuda_inc, *tool_src,
                           "-o", exe])
    subprocess.check_call([exe, out])


def build(verbose: bool = False) -> str:
    os.makedirs(BUILD, exist_ok=True)
    gen_tables()
    srcs = sources()
    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 1)) as ex:
        objs = list(ex.map(lambda s: _compile(s, verbose), srcs))
    stamp = LIB + ".objs"
    same_set = os.path.exists(stamp) and open(stamp).read() == "\n".join(objs)
    if not same_set or not os.path.exists(LIB) or os.path.getmtime(LIB) < max(os.path.getmtime(o) for o in objs):
        cmd = [nvcc(), *ARCH, "-shared", "-Xlinker", "--no-undefined", "-o", LIB, *objs, "-lcuda"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stderr}")
        with open(stamp, "w") as f:
            f.write("\n".join(objs))
    return LIB


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv))
