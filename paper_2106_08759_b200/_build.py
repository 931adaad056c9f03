"""Build libsntrup_gpu.so in-tree with nvcc for sm_100a (B200)."""
import os
import subprocess

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "libsntrup_gpu.so")
LIB_CHECKED = os.path.join(PKG, "libsntrup_gpu_check.so")   # bounds-checked build (tests only)
SOURCES = [os.path.join(CSRC, "sntrup_gpu.cu"), os.path.join(CSRC, "pool.cu")]
DEPS = SOURCES + [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cuh", ".h"))] + \
    [os.path.join(ROOT, "include", "sntrup_gpu.h")]

NVCC_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo", "-O3", "-std=c++17",
              "-Xcompiler", "-fPIC", "-shared", "-Xptxas", "-v"]


def needs_build() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(d) > t for d in DEPS)


def build_checked(force: bool = False) -> str:
    """The same library with device-side bounds checks (SNTRUP_CHECK) compiled in; load it by
    setting SNTRUP_GPU_LIB to its path (scripts/gpu_checked_tests.sh)."""
    return build(force, out=LIB_CHECKED, extra=["-DSNTRUP_BOUNDS_CHECK"])


def build(force: bool = False, verbose: bool = False, out: str = LIB, extra=()) -> str:
    target = out
    stale = not os.path.exists(target) or any(os.path.getmtime(d) > os.path.getmtime(target) for d in DEPS)
    if force or stale:
        nvcc = os.environ.get("NVCC", "nvcc")
        if not os.path.exists("/usr/local/cuda/bin/nvcc") and nvcc == "nvcc":
            pass
        elif nvcc == "nvcc":
            nvcc = "/usr/local/cuda/bin/nvcc"
        tmp = target + ".tmp%d" % os.getpid()
        cmd = [nvcc] + NVCC_FLAGS + list(extra) + ["-o", tmp] + SOURCES
        res = subprocess.run(cmd, capture_output=True, text=True)
        if res.returncode != 0:
            raise RuntimeError("nvcc failed:\n" + res.stderr[-6000:])
        if verbose:
            print(res.stderr)
        os.replace(tmp, target)
    return target


if __name__ == "__main__":
    build(force=True, verbose=True)
