"""Build librpd.so in-tree with nvcc for sm_100a (B200): every .cu compiled to an object in
parallel (separate translation units; host-side launchers link across them), then linked."""
import glob
import os
import subprocess
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
LIB = os.path.join(HERE, "librpd.so")
OBJ = os.path.join(HERE, "build")
SRCS = sorted(glob.glob(os.path.join(HERE, "csrc", "*.cu")))
HDRS = sorted(glob.glob(os.path.join(HERE, "csrc", "*.cuh"))) + \
    sorted(glob.glob(os.path.join(HERE, "csrc", "*.h"))) + [os.path.join(ROOT, "include", "rpd.h")]
DEPS = SRCS + HDRS

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
                     "-Xptxas", "-warn-spills"]


def stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(d) > t for d in DEPS)


def _objdir():
    """Objects live in a directory per flag set (variant builds do not mix with the default)."""
    import hashlib
    h = hashlib.sha1(" ".join(NVCC_FLAGS).encode()).hexdigest()[:10]
    return os.path.join(OBJ, h)


def _obj(src):
    return os.path.join(_objdir(), os.path.basename(src)[:-3] + ".o")


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not stale():
        return LIB
    nvcc = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
    os.makedirs(_objdir(), exist_ok=True)
    hdr_t = max(os.path.getmtime(h) for h in HDRS)

    def compile_one(src):
        o = _obj(src)
        if not force and os.path.exists(o) and os.path.getmtime(o) > max(hdr_t,
                                                                        os.path.getmtime(src)):
            return None
        tmp = o + f".{os.getpid()}.tmp.o"
        cmd = [nvcc, *NVCC_FLAGS, "-I", os.path.join(ROOT, "include"), "-c", "-o", tmp, src]
        r = subprocess.run(cmd, capture_output=not verbose, text=True)
        if r.returncode != 0:
            return f"nvcc failed on {os.path.basename(src)}:\n" + (r.stderr or "") + (r.stdout or "")
        os.replace(tmp, o)
        return None

    with ThreadPoolExecutor(max_workers=min(len(SRCS), os.cpu_count() or 4)) as ex:
        errs = [e for e in ex.map(compile_one, SRCS) if e]
    if errs:
        raise RuntimeError("\n".join(errs))
    tmp = LIB + f".{os.getpid()}.tmp"
    cmd = [nvcc, *ARCH, "-shared", "-o", tmp, *[_obj(s) for s in SRCS]]
    r = subprocess.run(cmd, capture_output=not verbose, text=True)
    if r.returncode != 0:
        raise RuntimeError("nvcc link failed:\n" + (r.stderr or "") + (r.stdout or ""))
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    print(build(force=True, verbose=True))
