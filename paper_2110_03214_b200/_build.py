"""Builds libmapa.so in-tree for sm_100a (nvcc cross-compiles without a GPU)."""
from __future__ import annotations

import os
import subprocess
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libmapa.so")
# translation units compiled in parallel
# (the per-width kernels in five parts each: see csrc/esa_w.cuh)
SOURCES = [os.path.join(CSRC, f"esa_w{w}_p{p}.cu") for w in (32, 16, 8) for p in range(5)] + \
    [os.path.join(CSRC, f) for f in ("esa_deep.cu", "esa.cu", "mapa_host.cpp")]
HEADERS = [os.path.join(CSRC, f) for f in ("internal.h", "esa_kernels.cuh", "esa_w.cuh")] + \
    [os.path.join(os.path.dirname(HERE), "include", "mapa.h")]

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-O3", "-std=c++17", "-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo",
         "-Xcompiler", "-fPIC", "-Xptxas", "-v"]
LINK = ["-gencode", "arch=compute_100a,code=sm_100a", "-Xcompiler", "-fPIC", "-shared", "-cudart", "static"]


def stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(s) > t for s in SOURCES + HEADERS)


def build(force: bool = False, verbose: bool = False) -> str:
    if force or stale():
        objdir = os.path.join(HERE, "build_obj")
        os.makedirs(objdir, exist_ok=True)
        objs = [os.path.join(objdir, os.path.basename(src) + ".o") for src in SOURCES]

        hdr_t = max(os.path.getmtime(h) for h in HEADERS)

        def compile_one(i):
            # incremental: an object is rebuilt when its source or any header is newer
            if not force and os.path.exists(objs[i]) and \
                    os.path.getmtime(objs[i]) > max(os.path.getmtime(SOURCES[i]), hdr_t):
                return None
            return subprocess.run([NVCC] + FLAGS + ["-c", "-o", objs[i], SOURCES[i]], capture_output=True, text=True)

        with ThreadPoolExecutor(min(len(SOURCES), max(2, os.cpu_count() or 2))) as ex:
            results = [r for r in ex.map(compile_one, range(len(SOURCES))) if r is not None]
        log = "".join(r.stderr for r in results)
        for r in results:
            if r.returncode != 0:
                raise RuntimeError("nvcc failed:\n" + r.stdout + r.stderr)
        r = subprocess.run([NVCC] + LINK + ["-o", LIB + ".tmp"] + objs, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError("nvcc link failed:\n" + r.stdout + r.stderr)
        if log:
            with open(os.path.join(HERE, "ptxas_info.txt"), "w") as f:
                f.write(log)
        os.replace(LIB + ".tmp", LIB)
        if verbose:
            print(log)
    return LIB


if __name__ == "__main__":
    build(force=True)
    print(LIB)
