"""Builds libchaos.so in-tree with nvcc for sm_100a (no JIT cache, so the .so travels with the repo)."""
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
SRC = [os.path.join(HERE, "csrc", "chaos_runtime.cu")]
DEPS = SRC + [os.path.join(HERE, "csrc", "chaos_kernels.cuh"), os.path.join(ROOT, "include", "chaos.h")]
OUT = os.path.join(HERE, "libchaos.so")
# instrumented variant (per-phase clock64 timing, chaos_debug_phase_times); profiling only
OUT_TIMING = os.path.join(HERE, "libchaos_timing.so")
NVCC_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
              "-Xcompiler", "-fPIC", "-shared", "-diag-suppress", "550,177"]


def build(force=False, verbose=False, timing=False):
    out = OUT_TIMING if timing else OUT
    if not force and os.path.exists(out) and os.path.getmtime(out) >= max(os.path.getmtime(p) for p in DEPS):
        return out
    cmd = ["nvcc", *NVCC_FLAGS, "-I" + os.path.join(ROOT, "include"), "-o", out, *SRC]
    if timing:
        cmd.insert(1, "-DCHAOS_TIMING")
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
    subprocess.check_call(cmd)
    return out


def build_variant(name, defs=(), timing=False, only_net=None):
    """A/B experiments: libchaos_<name>.so with extra -D definitions (optionally one net only,
    CHAOS_ONLY_NET: ~4x faster to compile).  Load it with CHAOS_LIB=<path>."""
    out = os.path.join(HERE, f"libchaos_{name}.so")
    cmd = ["nvcc", *NVCC_FLAGS, "-I" + os.path.join(ROOT, "include"), "-o", out, *SRC]
    extra = [f"-D{d}" for d in defs]
    if timing:
        extra.append("-DCHAOS_TIMING")
    if only_net:
        extra += ["-DCHAOS_ONLY_NET", f"-DCHAOS_ONLY_NET_{only_net}=1"]
    subprocess.check_call(cmd[:1] + extra + cmd[1:])
    return out


if __name__ == "__main__":
    import sys
    build(force="--force" in sys.argv, verbose="-v" in sys.argv, timing="--timing" in sys.argv)
