"""Build the native library in-tree with nvcc for sm_100a.

`python -m paper_1110_2561_b200._build` (or `__graft_entry__.build()`)
compiles csrc/*.cu + csrc/*.cpp into paper_1110_2561_b200/libisingdos_b200.so.
The CUDA runtime is linked statically, so the .so only needs the driver on
the GPU box.
"""

import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "libisingdos_b200.so")
# bounds-checked variant (traps on an out-of-histogram address); load it with
# ISD_LIBRARY=<path> — the stand-in for compute-sanitizer (closed on the pool)
LIB_DEBUG = os.path.join(PKG, "libisingdos_b200_dbg.so")

SOURCES = ["plan.cpp", "enumerate.cu", "thermo.cu", "calibrate.cu", "capi.cu",
           "jit.cpp", "knobs.cpp", "cache.cpp", "naive.cu"]
HEADERS = ["isd_internal.h", "k1_body.cuh"]

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC,-O3,-Wall",
    "-shared",
]


def nvcc_path() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    return "nvcc"


def _inputs():
    files = [os.path.join(CSRC, s) for s in SOURCES + HEADERS]
    files.append(os.path.join(ROOT, "include", "isingdos_b200.h"))
    return files


def up_to_date(lib: str = LIB) -> bool:
    if not os.path.exists(lib):
        return False
    t = os.path.getmtime(lib)
    return all(os.path.getmtime(f) <= t for f in _inputs())


def _embed_body() -> None:
    """csrc/k1_body_str.inc: k1_body.cuh as a C++ raw string (for NVRTC)."""
    body = open(os.path.join(CSRC, "k1_body.cuh")).read()
    assert ")ISDBODY\"" not in body
    text = 'R"ISDBODY(' + body + ')ISDBODY"\n'
    path = os.path.join(CSRC, "k1_body_str.inc")
    if not os.path.exists(path) or open(path).read() != text:
        with open(path, "w") as f:
            f.write(text)


def build(force: bool = False, verbose: bool = False,
          debug: bool = False) -> str:
    lib = LIB_DEBUG if debug else LIB
    if not force and up_to_date(lib):
        return lib
    _embed_body()
    # one nvcc per source, in parallel, then one link
    tag = "dbg" if debug else "rel"
    objdir = os.path.join(PKG, "_obj", tag)
    os.makedirs(objdir, exist_ok=True)
    compile_flags = [f for f in NVCC_FLAGS if f != "-shared"]
    extra = (["-DISD_DEBUG_BOUNDS"] if debug else []) + \
        (["-Xptxas=-v"] if verbose else [])

    # the on-disk plan / cubin cache keys carry a hash of the sources, so a
    # rebuilt library never reads another build's entries
    import hashlib
    h = hashlib.sha256()
    for f in _inputs():
        h.update(os.path.basename(f).encode())
        h.update(open(f, "rb").read())
    extra.append(f"-DISD_BUILD_ID=\"{h.hexdigest()[:16]}{'-dbg' if debug else ''}\"")

    def compile_one(unit):
        src, defines, name = unit
        obj = os.path.join(objdir, name + ".o")
        cmd = [nvcc_path(), *extra, *defines, *compile_flags, "-I",
               os.path.join(ROOT, "include"), "-c", os.path.join(CSRC, src),
               "-o", obj]
        if verbose:
            print(" ".join(cmd), flush=True)
        subprocess.run(cmd, check=True)
        return obj

    # enumerate.cu holds the hoisted kernel's 64 instantiations: compiled as
    # four translation units (ISD_HOIST_PART, two class counts each)
    units = []
    for src in SOURCES:
        stem = os.path.splitext(src)[0]
        if src == "enumerate.cu":
            units += [(src, [f"-DISD_HOIST_PART={p}"], f"{stem}_{p}")
                      for p in range(4)]
        else:
            units.append((src, [], stem))
    from concurrent.futures import ThreadPoolExecutor
    with ThreadPoolExecutor(max_workers=len(units)) as pool:
        objs = list(pool.map(compile_one, units))
    cmd = [nvcc_path(), "-gencode", "arch=compute_100a,code=sm_100a",
           "-shared", *objs, "-ldl", "-o", lib + ".tmp"]
    subprocess.run(cmd, check=True)
    os.replace(lib + ".tmp", lib)
    return lib


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv,
                debug="--debug" in sys.argv))
