"""Build libmuxflow.so in-tree with nvcc for sm_100a (no torch extension
machinery: the library is plain C ABI over the CUDA runtime)."""

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
OUT = os.path.join(HERE, "libmuxflow.so")
SOURCES = ("api.cu", "score.cu", "auction.cu", "ssp.cu", "ssp_w64.cu", "canon.cu", "mlp.cu")
HEADERS = ("common.cuh",)
NVCC_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
              "-Xcompiler", "-fPIC", "-shared", "-Xptxas", "-v"]


def _stale():
    if not os.path.exists(OUT):
        return True
    t = os.path.getmtime(OUT)
    deps = [os.path.join(CSRC, f) for f in SOURCES + HEADERS]
    deps.append(os.path.join(HERE, "..", "include", "muxflow.h"))
    return any(os.path.getmtime(d) > t for d in deps)


OBJDIR = os.path.join(HERE, "build")


def _compile(nvcc, src, obj, force, extra=()):
    """One translation unit -> object (skipped when the object is newer than
    the source and the shared headers)."""
    deps = [src, os.path.join(CSRC, "common.cuh"), os.path.join(HERE, "..", "include", "muxflow.h")]
    if os.path.basename(src) == "ssp_w64.cu":   # compiles ssp.cu a second time (int64 weights)
        deps.append(os.path.join(CSRC, "ssp.cu"))
    if not force and os.path.exists(obj) and all(os.path.getmtime(d) <= os.path.getmtime(obj) for d in deps):
        return None
    flags = [f for f in NVCC_FLAGS if f != "-shared"] + list(extra)
    return subprocess.Popen([nvcc] + flags + ["-c", src, "-o", obj], stdout=subprocess.PIPE,
                            stderr=subprocess.PIPE, text=True)


def build(force=False, verbose=False, extra=(), out=None, objdir=None):
    """Build the library; `extra` nvcc flags with their own `out` / `objdir`
    give experiment variants (tools/build_variant.py)."""
    out = out or OUT
    objdir = objdir or OBJDIR
    if not force and not extra and not _stale():
        return OUT
    nvcc = os.environ.get("NVCC", "nvcc")
    os.makedirs(objdir, exist_ok=True)
    objs, procs = [], []
    for f in SOURCES:
        obj = os.path.join(objdir, f.replace(".cu", ".o"))
        objs.append(obj)
        p = _compile(nvcc, os.path.join(CSRC, f), obj, force, extra)
        if p is not None:
            procs.append((f, p))
    for f, p in procs:   # translation units compile in parallel
        so, se = p.communicate()
        if p.returncode != 0:
            sys.stderr.write(so + se)
            raise RuntimeError(f"nvcc failed compiling {f}")
        if verbose:
            sys.stderr.write(se)
    cmd = [nvcc, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-Xcompiler", "-fPIC",
           "-o", out + ".tmp"] + objs
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError("nvcc failed linking libmuxflow.so")
    os.replace(out + ".tmp", out)
    return out


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
