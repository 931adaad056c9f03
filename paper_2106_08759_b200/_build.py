"""Build libsntrup_gpu.so in-tree with nvcc for sm_100a (B200).

One translation unit per parameter set (csrc/ps_<p>.cu) plus the C ABI (capi.cu) and the key
pool (pool.cu), compiled in parallel and linked into one shared library."""
import concurrent.futures as cf
import os
import subprocess

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "libsntrup_gpu.so")
LIB_CHECKED = os.path.join(PKG, "libsntrup_gpu_check.so")   # bounds-checked build (tests only)
LIB_TRACE = os.path.join(PKG, "libsntrup_gpu_trace.so")     # role-timing build (scripts/ws_trace.py)
OBJDIR = os.path.join(PKG, "build")
SOURCES = [os.path.join(CSRC, f) for f in
           ("capi.cu", "ps_761.cu", "ps_1277.cu", "ps_1013.cu", "ps_953.cu", "ps_857.cu", "ps_653.cu", "pool.cu",
            "probe_split.cu")]
DEPS = SOURCES + [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cuh", ".h"))] + \
    [os.path.join(ROOT, "include", "sntrup_gpu.h")]

NVCC_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo", "-O3", "-std=c++17",
              "-Xcompiler", "-fPIC", "-Xptxas", "-v"]


def _nvcc():
    nvcc = os.environ.get("NVCC", "nvcc")
    if nvcc == "nvcc" and os.path.exists("/usr/local/cuda/bin/nvcc"):
        nvcc = "/usr/local/cuda/bin/nvcc"
    return nvcc


def needs_build() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(d) > t for d in DEPS)


def build_checked(force: bool = False) -> str:
    """The same library with device-side bounds checks (SNTRUP_CHECK) compiled in; load it by
    setting SNTRUP_GPU_LIB to its path (scripts/gpu_checked_tests.sh)."""
    return build(force, out=LIB_CHECKED, extra=["-DSNTRUP_BOUNDS_CHECK"])


def build_trace(force: bool = False) -> str:
    """The library with the warp-specialised kernels' role timing compiled in (SNTRUP_WS_TRACE)."""
    return build(force, out=LIB_TRACE, extra=["-DSNTRUP_WS_TRACE"])


def build(force: bool = False, verbose: bool = False, out: str = LIB, extra=()) -> str:
    target = out
    stale = not os.path.exists(target) or any(os.path.getmtime(d) > os.path.getmtime(target) for d in DEPS)
    if not (force or stale):
        return target
    nvcc = _nvcc()
    tag = {(): "rel", ("-DSNTRUP_BOUNDS_CHECK",): "chk"}.get(tuple(extra), "trc")
    os.makedirs(OBJDIR, exist_ok=True)

    def compile_one(src):
        obj = os.path.join(OBJDIR, "%s_%s.o" % (os.path.basename(src)[:-3], tag))
        tmp = obj + ".tmp%d" % os.getpid()
        cmd = [nvcc] + NVCC_FLAGS + list(extra) + ["-c", "-o", tmp, src]
        res = subprocess.run(cmd, capture_output=True, text=True)
        if res.returncode != 0:
            raise RuntimeError("nvcc failed on %s:\n%s" % (os.path.basename(src), res.stderr[-6000:]))
        os.replace(tmp, obj)
        return obj, res.stderr

    with cf.ThreadPoolExecutor(max_workers=max(1, min(len(SOURCES), os.cpu_count() or 1))) as ex:
        results = list(ex.map(compile_one, SOURCES))
    if verbose:
        for _, err in results:
            print(err)
    tmp = target + ".tmp%d" % os.getpid()
    res = subprocess.run([nvcc, "-shared", "-o", tmp] + [o for o, _ in results], capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError("link failed:\n" + res.stderr[-6000:])
    os.replace(tmp, target)
    return target


if __name__ == "__main__":
    build(force=True, verbose=True)
