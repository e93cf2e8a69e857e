"""In-tree build of libdashcu.so for sm_100a (explicit nvcc; no JIT cache).

    python -m paper_2505_17218_b200.build        # or __graft_entry__.build()
"""
from __future__ import annotations

import concurrent.futures as cf
import hashlib
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
OUT_DIR = os.path.join(PKG, "lib")
OBJ_DIR = os.path.join(OUT_DIR, "obj")
# Experiment builds (A/B of compile-time variants, tools only): DASHCU_NVCC_EXTRA adds nvcc
# flags (e.g. -D...), DASHCU_LIB_OUT names the output library; load it with DASHCU_LIB_PATH.
LIB = os.environ.get("DASHCU_LIB_OUT") or os.path.join(OUT_DIR, "libdashcu.so")
# object list of each built library (untracked; lives beside the objects)
OBJS_LIST = os.path.join(OBJ_DIR, os.path.basename(LIB) + ".objs")

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC,-fvisibility=hidden", "--expt-relaxed-constexpr",
         "-Xptxas", "-v" if os.environ.get("DASHCU_PTXAS_V") else "-O3", f"-I{os.path.join(ROOT, 'include')}"]
FLAGS += os.environ.get("DASHCU_NVCC_EXTRA", "").split()


def sources():
    return sorted(os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith(".cu"))


def _headers_digest():
    h = hashlib.sha1()
    for f in sorted(os.listdir(CSRC)):
        if f.endswith((".cuh", ".h")):
            h.update(open(os.path.join(CSRC, f), "rb").read())
    h.update(open(os.path.join(ROOT, "include", "dashcu.h"), "rb").read())
    h.update(" ".join(ARCH + FLAGS).encode())
    return h.hexdigest()[:12]


def _compile(src, dig):
    obj = os.path.join(OBJ_DIR, os.path.basename(src) + f".{dig}.o")
    if os.path.exists(obj) and os.path.getmtime(obj) >= os.path.getmtime(src):
        return obj, ""
    cmd = [NVCC, *ARCH, *FLAGS, "-c", src, "-o", obj]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{r.stderr}")
    return obj, r.stderr


def build(verbose: bool = False) -> str:
    os.makedirs(OBJ_DIR, exist_ok=True)
    dig = _headers_digest()
    srcs = sources()
    with cf.ThreadPoolExecutor(max_workers=min(8, len(srcs))) as ex:
        res = list(ex.map(lambda s: _compile(s, dig), srcs))
    objs = [o for o, _ in res]
    if verbose:
        for _, log in res:
            if log:
                print(log, file=sys.stderr)
    newest = max(os.path.getmtime(o) for o in objs)
    if not os.path.exists(LIB) or os.path.getmtime(LIB) < newest or _stale_objs(objs):
        # --no-undefined: a symbol left undefined (e.g. given internal linkage by mistake)
        # must fail here, not at dlopen time on the GPU box
        cmd = [NVCC, *ARCH, "-shared", "-Xlinker", "--no-undefined", "-o", LIB, *objs, "-lcudart", "-ldl"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stderr}")
        with open(OBJS_LIST, "w") as f:
            f.write("\n".join(objs))
    _prune_objs()
    return LIB


def _prune_objs():
    """Drop object files no library's .objs list references (old header digests)."""
    keep = set()
    for f in os.listdir(OBJ_DIR):
        if f.endswith(".objs"):
            with open(os.path.join(OBJ_DIR, f)) as fh:
                keep.update(os.path.abspath(ln.strip()) for ln in fh if ln.strip())
    for f in os.listdir(OBJ_DIR):
        p = os.path.abspath(os.path.join(OBJ_DIR, f))
        if f.endswith(".o") and p not in keep:
            os.remove(p)


def _stale_objs(objs):
    try:
        return open(OBJS_LIST).read().split("\n") != objs
    except OSError:
        return True


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv))
